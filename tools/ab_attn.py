#!/usr/bin/env python
"""A/B timing of the attention kernel across sequence lengths (one JSON line per case).

Kernel variants are selected by environment variables read at launch (e.g. FPB_FA_GS), so run
this once per variant:  FPB_FA_GS=1 python tools/ab_attn.py
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import workload  # noqa: E402
from tools.configs import timed  # noqa: E402

D = 128


def plan_flops(plan, M):
    c = plan.counts.to(torch.int64).sum().item()
    ndiag = plan.counts.numel()  # every max-threshold row keeps its diagonal block
    return (c - ndiag) * 4.0 * D * 128 * 128 + ndiag * 4.0 * D * 128 * 129 / 2, c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default=os.environ.get("FPB_FA_GS", "auto"))
    ap.add_argument("--cases", default="32768:0.12,131072:0.02,131072:0.12,262144:0.12")
    ap.add_argument("--dense", default="32768,131072")
    args = ap.parse_args()
    cache = {}
    dense_L = {int(x) for x in args.dense.split(",") if x}
    for case in args.cases.split(","):
        L, a = case.split(":")
        L, a = int(L), float(a)
        if L not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[L] = workload.composite(5, 1, 32, 4, L, device="cuda")
        q, k, v = cache[L]
        grid = fp.make_block_grid(L, 128)
        tau = 1 / math.sqrt(D)
        # device time of each stage from CUDA-graph replays (no host work in the timed region)
        r = fp.PrefillRunner(q, k, v, fp.PipelineConfig(alpha=a)).capture()
        td = timed(r.replay_discover, reps=3, warm=1)
        t = timed(r.replay_attend, reps=3, warm=1)
        r.check()
        plan = r.plan
        fl, visits = plan_flops(plan, grid.num_query_blocks)
        rec = dict(tag=args.tag, L=L, alpha=a, visits=visits, disc_ms=td, attn_ms=t,
                   tflops=fl / t / 1e9, ns_per_visit=t * 1e6 / visits)
        if L in dense_L:
            td = timed(lambda: fp.dense_attention(q, k, v, tau), reps=2, warm=1)
            rec["dense_ms"] = td
            rec["dense_tflops"] = 4.0 * D * 32 * L * (L + 1) / 2 / td / 1e9
            dense_L.discard(L)
        print(json.dumps(rec), flush=True)
        del plan


if __name__ == "__main__":
    main()
