#!/usr/bin/env python
"""Cycle accounting of discover_kernel (build with -DFPB_TRACE, load via FPB200_LIB)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import _abi, workload  # noqa: E402

NAMES = {0: "epi wait accumulator", 1: "epi TMEM load", 2: "epi chunk max/exp2/sum",
         3: "epi first barrier", 16: "epi rescaled energies + 2nd barrier",
         17: "epi threshold + ballots + 3rd barrier", 18: "epi compaction (active idx stores)",
         4: "epi fill (idx = N) + counts", 5: "epi wait item",
         8: "mma wait Q", 9: "mma wait accumulator free", 10: "mma wait kbar chunk",
         11: "mma issue", 12: "producer item ring full", 13: "producer Q buffer busy",
         14: "producer kbar ring full", 15: "producer atomic", 19: "mma wait item", 21: "mma item decode", 22: "mma chunk loop overhead",
         20: "kernel cycles (CTA, MMA warp lane 0)",
         6: "in-kernel pooling: launch -> prologue end (CTA)",
         23: "producer wait pooled kbar chunk",
         24: "pool: claim + issue (per warp)", 25: "pool: wait rows (per warp)",
         26: "pool: channel sums (per warp)", 27: "pool: stores + fences + release (per warp)"}
PER_SM = {6}
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = workload.composite(5, 1, 32, 4, L, device="cuda")
cfg = fp.PipelineConfig()
lib = _abi.lib()
buf = (C.c_ulonglong * 32)()
for _ in range(2):
    fp.discover_select(q, k, cfg)
torch.cuda.synchronize()
lib.fpb_dtrace_read(buf, 1)
plan = fp.discover_select(q, k, cfg)[0]
torch.cuda.synchronize()
lib.fpb_dtrace_read(buf, 1)
M = (L + 127) // 128
items = 32 * M
chunks = 32 * sum(I // 128 + 1 for I in range(M))
epi_warps = 148 * 8
print(f"L={L}: items {items}, chunks {chunks}; per-SM totals in Kcycles (epilogue: per warp avg)")
if buf[29]:
    t0 = (~buf[28]) & (2**64 - 1)
    print(f"CTA start spread {(buf[29] - t0) / 1e3:.2f} us; latest prologue end +{(buf[30] - t0) / 1e3:.2f} us; "
          f"latest chunk acquire +{(buf[31] - t0) / 1e3:.2f} us (globaltimer, from the first CTA start)")
for i, n in NAMES.items():
    if i >= 24:
        per_sm = buf[i] / (148 * 12) / 1e3  # average per warp (12 pooling warps per CTA)
    elif (i < 8 or 16 <= i <= 18) and i not in PER_SM:
        per_sm = buf[i] / epi_warps / 1e3  # average per epilogue warp
    else:
        per_sm = buf[i] / 148 / 1e3
    epi = (i < 8 or 16 <= i <= 18) and i not in PER_SM
    print(f"{n:40s} {per_sm:10.1f} Kcyc per {'epilogue warp' if epi else 'SM'}")
