"""Top CUDA source lines by warp-stall samples from an ncu report (needs -lineinfo).
Usage: python tools/ncu_lines.py REPORT.ncu-rep [substring-of-file] [N]"""
import csv
import io
import subprocess
import sys


def main(rep, filt="", top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur_file, res = "", []
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] not in ("",) and len(r) > 5 and r[0].isdigit():
            try:
                res.append((int(r[4]), cur_file.split("/")[-1], int(r[0]), r[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(x[0] for x in res) or 1
    print(f"total samples {tot}")
    for s, f, ln, src in sorted((x for x in res if filt in x[1]), reverse=True)[:top]:
        print(f"{s:7d} {100 * s / tot:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 30)
