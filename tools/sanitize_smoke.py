#!/usr/bin/env python
"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): discovery with in-kernel pooling (two-pass and fused epilogue), selection,
block-sparse and dense attention (bf16 and fp32 inputs), KV-range phases, row shards, the SIMT
path and the host pipeline."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06199_b200 as fp  # noqa: E402

cfg = fp.PipelineConfig()
for (Z, Hq, Hkv, L) in [(1, 2, 1, 1000), (2, 4, 2, 2300)]:
    q, k, v = (x.cuda() for x in fp.workload.composite(5, Z, Hq, Hkv, L))
    grid = fp.make_block_grid(L, 128)
    tau = cfg.resolved_scale(128)
    plan, _, _ = fp.discover_select(q, k, cfg)
    fp.discover(q, k, grid, tau)
    fp.block_sparse_attention(q, k, v, plan, grid, tau)
    fp.dense_attention(q, k, v, tau)
    rows = fp.shard.zigzag_shard(2, 1)
    p2, _, _ = fp.discover_select(q, k, cfg, rows=rows)
    fp.block_sparse_attention(q, k, v, p2, grid, tau, rows=rows)
    qf, kf, vf = (x.float() for x in (q, k, v))
    pf, _, _ = fp.discover_select(qf, kf, cfg)
    fp.block_sparse_attention(qf, kf, vf, pf, grid, tau)
# fused epilogue (>= 1024 key blocks); run with FPB_FA_PHASES=2 to force KV-range phases

q, k, v = (x.cuda() for x in fp.workload.composite(7, 1, 1, 1, 1024 * 128 + 77))
plan, _, _ = fp.discover_select(q, k, cfg)
fp.block_sparse_attention(q, k, v, plan, fp.make_block_grid(q.shape[2], 128), cfg.resolved_scale(128))
# SIMT path (d = 64)
q, k, v = (torch.randn(1, 2, 500, 64, device="cuda") for _ in range(3))
c64 = fp.PipelineConfig(block_size=64, sink_tokens=64, window_tokens=64)
p64, _, _ = fp.discover_select(q, k, c64)
fp.block_sparse_attention(q, k, v, p64, fp.make_block_grid(500, 64), c64.resolved_scale(64))
# host pipeline
q, k, v = fp.workload.composite(9, 1, 4, 2, 3000)
out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()
fp.prefill_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), cfg, out, lse)
torch.cuda.synchronize()
print("sanitize smoke done")
