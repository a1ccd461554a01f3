"""Where a kernel's no-instruction (instruction fetch) stalls sit: SASS address ranges with the most
stall_no_inst samples, with the CUDA source line of the first instruction of each 256-byte block.
Usage: python tools/ncu_noinst.py REPORT.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hdr = rows[1]
    ia, ino, isrc = hdr.index("Address"), hdr.index("stall_no_inst"), hdr.index("Source")
    blocks = collections.Counter()
    first = {}
    tot = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        a = int(r[ia], 16)
        v = int(r[ino] or 0)
        tot += v
        blocks[a // 256] += v
        first.setdefault(a // 256, r[isrc].strip())
    print(f"total no_inst samples {tot}")
    for b, v in blocks.most_common(top):
        print(f"{v:6d}  0x{b * 256:x}  {first[b][:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
