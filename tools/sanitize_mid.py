#!/usr/bin/env python
"""Mid-size racecheck input for compute-sanitizer (8K with 8 Q / 2 KV heads; 140 key blocks):
two-pass discovery, maps, attention.  usage: compute-sanitizer --tool racecheck python tools/sanitize_mid.py"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2603_06199_b200 as fp
cfg = fp.PipelineConfig()
for L, H, Hk in [(8192, 8, 2), (140 * 128, 2, 1)]:
    q, k, v = (x.cuda() for x in fp.workload.composite(11, 1, H, Hk, L))
    plan, _, _ = fp.discover_select(q, k, cfg)
    m = fp.discover(q, k, fp.make_block_grid(L, 128), cfg.resolved_scale(128))
    fp.block_sparse_attention(q, k, v, plan, fp.make_block_grid(L, 128), cfg.resolved_scale(128))
torch.cuda.synchronize(); print("mid done")
