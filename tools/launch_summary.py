#!/usr/bin/env python
"""Aggregates an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel name: launches, total and mean time, share.
Usage: python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import sys

UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
        "second": 1.0}


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        for r in csv.reader(f):
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr is None or len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            t = float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]]
            k = d["Kernel Name"].split("(")[0].replace("void ", "")
            agg[k][0] += 1
            agg[k][1] += t
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    print(f"{n} launches, {tot:.4f} s kernel time")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k[:60]:60s} {c:7d} {t:9.4f} s {1e6 * t / c:9.1f} us {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()
