"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys


def main(path):
    hdr = None
    agg = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:64]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in agg.items():
        print(f"{k:64s} {n:4d} {t / 1e3:10.3f} ms  {t / n:10.1f} us each  {100 * t / tot:5.1f}%")
    print(f"{'total':64s}      {tot / 1e3:10.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
