"""Text summary of one ncu --set full report (first kernel): headline counters,
warp-stall breakdown and the SASS instructions with the most stall samples.
Usage: python tools/ncu_report.py REPORT.ncu-rep > profiles/NAME.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    print(f"# ncu --set full summary: {rep.split('/')[-1]}")
    print(f"kernel: {d.get('Kernel Name', '?')}")
    for k in KEYS:
        if k in d:
            print(f"  {k:72s} {d[k]:>14s} {u.get(k, '')}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    print("\nwarp stall samples (all):")
    for v, k in sorted(st, reverse=True)[:12]:
        print(f"  {k:28s} {v:8.0f}  {100 * v / tot:5.1f}%")
    lines = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    h = lines[1]
    i_src, i_smp = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    ins = []
    for r in lines[2:]:
        try:
            ins.append((int(r[i_smp]), r[0], r[i_src].strip()))
        except (ValueError, IndexError):
            pass
    print("\ntop SASS instructions by stall samples:")
    for s, a, src in sorted(ins, reverse=True)[:25]:
        print(f"  {s:6d}  {a[-6:]}  {src}")


if __name__ == "__main__":
    main(sys.argv[1])
