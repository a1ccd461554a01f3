"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "")
                v = float(d["Metric Value"].replace(",", ""))
                unit = d["Metric Unit"]
                v = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
                out.append((name, v, d.get("Grid Size", "")))
    return out


if __name__ == "__main__":
    for path in sys.argv[1:]:
        L = load(path)
        agg = collections.OrderedDict()
        for name, us, grid in L:
            a = agg.setdefault(name, [0, 0.0, grid])
            a[0] += 1
            a[1] += us
        tot = sum(v[1] for v in agg.values())
        print(f"== {path}: {len(L)} launches, {tot:.1f} us total")
        for name, (cnt, us, grid) in agg.items():
            print(f"  {name:45s} n={cnt:4d} avg={us/cnt:9.2f} us  share={100*us/tot:5.1f}%  grid={grid}")
