#!/usr/bin/env python
"""One FlashPrefill step on one synthetic Qwen3 layer, for ncu captures of a given length.

The inputs are exactly those of bench.py's `sweep` entries (workload.composite seed 5, generated on
the GPU) or, with --bench-inputs, bench.py's headline layer (seed 1234, generated on the CPU), so a
capture's DRAM bytes can be filed in profiles/ncu_traffic.json under the config bench.py looks up.
Warm-up launches run first; then `--reps` plain (non-graph) discover+select and attention calls.

usage: ncu ... python tools/ncu_step.py --L 262144 [--reps 1] [--bench-inputs]
"""
from __future__ import annotations

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=0.12)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--bench-inputs", action="store_true")
    a = ap.parse_args()
    if a.bench_inputs:
        q, k, v = (x.cuda() for x in workload.composite(1234, 1, a.hq, a.hkv, a.L)) 
    else:
        q, k, v = workload.composite(5, 1, a.hq, a.hkv, a.L, device="cuda")
    cfg = fp.PipelineConfig(alpha=a.alpha)
    r = fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16)
    for _ in range(a.warmup + a.reps):
        r.discover()
        r.attend()
    torch.cuda.synchronize()
    print(f"L={a.L} visits={r.check()}")


if __name__ == "__main__":
    main()
