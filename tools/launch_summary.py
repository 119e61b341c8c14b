#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list: per kernel
name, launches and mean / total duration (us), in first-launch order.

usage: python tools/launch_summary.py gpurun_out/x_launches.csv [--skip N]"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1 + skip:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[ui]]
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.replace("void ", "")
        name = name.split("(")[0].split("<")[0].split("::")[-1]
        v = float(r[vi].replace(",", "")) * scale
        n, tot = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, tot + v)
    for name, (n, tot) in agg.items():
        print(f"{name:40s} {n:5d} launches  mean {tot / n:10.2f} us  total {tot:10.1f} us")


if __name__ == "__main__":
    main()
