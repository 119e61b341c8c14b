#!/usr/bin/env python
"""Cycle accounting of fa2_kernel (build with -DFPB_TRACE, load via FPB200_LIB)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import _abi, workload  # noqa: E402

# index -> (name, normaliser): v = per visit per warp (8 softmax warps), V = per visit (1 warp),
# i = per item per warp (4 epilogue warps), I = per item (1 warp)
NAMES = {0: ("softmax wait S", "v"), 1: ("softmax S ld + max", "v"), 2: ("softmax max agree", "v"),
         3: ("softmax exp2 + pack", "v"), 4: ("softmax wait P buffer", "v"),
         5: ("softmax P store + arrive", "v"), 7: ("mma wait Q", "I"), 8: ("mma wait S free", "V"),
         9: ("mma wait K", "V"), 10: ("mma wait O free", "I"), 11: ("mma wait V", "V"),
         12: ("mma wait P half0", "V"), 13: ("mma wait P half1", "V"),
         14: ("producer wait ring", "V"), 15: ("epi wait stats", "i"), 16: ("epi wait O", "i"),
         17: ("epi O ld+norm+stage", "i"), 18: ("epi TMA store", "i"), 19: ("kernel (warp 1)", "c")}
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = (x.cuda() for x in workload.qwen3_30b_a3b(L, seed=1234))
cfg = fp.PipelineConfig()
plan = fp.discover_select(q, k, cfg)[0]
grid = fp.make_block_grid(L, 128)
lib = _abi.lib()
buf = (C.c_ulonglong * 24)()
for _ in range(2):
    fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128))
torch.cuda.synchronize()
lib.fpb_trace2_read(buf, 1)
fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128))
torch.cuda.synchronize()
lib.fpb_trace2_read(buf, 1)
visits = int(plan.counts.sum())
items = q.shape[1] * grid.num_query_blocks
ctas = 148
print(f"L={L} visits={visits} items={items}; per-CTA visits {visits / ctas:.0f}")
for i, (n, kind) in NAMES.items():
    den = {"v": 8 * visits, "V": visits, "i": 4 * items, "I": items, "c": ctas}[kind]
    print(f"{n:26s} total {buf[i] / 1e6:10.2f} Mcyc   per unit {buf[i] / den:10.1f}  ({kind})")
print(f"kernel cycles per visit per CTA: {buf[19] / ctas / (visits / ctas):.1f}")
