#!/usr/bin/env python
"""Cycle accounting of fa_kernel (build variant with -DFPB_TRACE, load via FPB200_LIB)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import _abi, workload  # noqa: E402

NAMES = {0: "softmax wait S", 1: "softmax ld+max", 2: "softmax rescale", 3: "softmax exp half0",
         4: "softmax exp half1", 5: "softmax epilogue (per item)", 8: "mma wait V",
         9: "mma wait P half0", 10: "mma wait P half1", 11: "mma wait K",
         12: "producer wait ring slot", 13: "producer wait Q tile (per item)",
         14: "producer wait scheduler (per item)", 15: "mma wait Q (per item)"}
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = (x.cuda() for x in workload.qwen3_30b_a3b(L, seed=1234))
cfg = fp.PipelineConfig()
plan = fp.discover_select(q, k, cfg)[0]
grid = fp.make_block_grid(L, 128)
lib = _abi.lib()
buf = (C.c_ulonglong * 16)()
for _ in range(2):
    fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128))
torch.cuda.synchronize()
lib.fpb_trace_read(buf, 1)
fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128))
torch.cuda.synchronize()
lib.fpb_trace_read(buf, 1)
visits = int(plan.counts.sum())
items = q.shape[1] * grid.num_query_blocks
for i, n in NAMES.items():
    per = (buf[i] / (4 * visits) if i < 5 else buf[i] / (4 * items) if i == 5
           else buf[i] / items if i in (13, 14, 15) else buf[i] / visits)
    print(f"{n:32s} total {buf[i]/1e6:10.2f} Mcyc   per block-visit {per:8.1f} cyc"
          + ("  (per warp)" if i < 5 else ("  (per item per warp)" if i == 5 else "")))
