"""Per-launch list (duration, DRAM read / write) from an ncu CSV taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.
Usage: python tools/ncu_launches.py LAUNCHES.csv [name-substring ...]"""
import collections
import csv
import sys


def to_us(v, unit):
    return v / 1000.0 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1000.0


def to_mb(v, unit):
    return {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6) * v


def main(path, filt):
    hdr, launches = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        L = launches.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", "")})
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Name"] == "gpu__time_duration.sum":
            L["us"] = to_us(v, d["Metric Unit"])
        elif d["Metric Name"] == "dram__bytes_read.sum":
            L["rd"] = to_mb(v, d["Metric Unit"])
        elif d["Metric Name"] == "dram__bytes_write.sum":
            L["wr"] = to_mb(v, d["Metric Unit"])
    for i, L in launches.items():
        if filt and not any(f in L["name"] for f in filt):
            continue
        print(f"{int(i):4d} {L['name'][-60:]:60s} {L.get('us', 0):9.1f} us  read {L.get('rd', 0):8.1f} MB  write {L.get('wr', 0):7.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
