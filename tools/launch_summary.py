"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: total us per kernel."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}


def main(path):
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} us {100 * t / tot:5.1f}% {c:5d}x  {k}")
    print(f"{tot:10.1f} us total")


if __name__ == "__main__":
    main(sys.argv[1])
