#!/usr/bin/env python
"""Warp-stall samples per CUDA source line from an ncu report (needs -lineinfo + --import-source).

usage: python tools/ncu_lines.py report.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iss = h.index("Warp Stall Sampling (All Samples)")
per = defaultdict(float)
src = {}
cur = None
for r in rows[hi + 1:]:
    if len(r) <= iss:
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else r[0]
        src[cur] = r[1]
    try:
        per[cur] += float(r[iss] or 0)
    except ValueError:
        pass
tot = sum(per.values()) or 1
print(f"total samples {tot:.0f}")
for ln, v in sorted(per.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:7.0f} {100 * v / tot:5.1f}%  L{ln}: {src.get(ln, '').strip()[:100]}")
