#!/usr/bin/env python
"""Timeline of fpb_host_prefill (the e2e call bench.py times) at the bench workload.

Run with FPB_E2E_TRACE=1 so the library prints per-chunk H2D / kernel / D2H completion times.
usage: FPB_E2E_TRACE=1 python tools/e2e_trace.py [--L 32768]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    q, k, v = workload.qwen3_30b_a3b(args.L, seed=1234, device="cuda")
    qp, kp, vp = (x.cpu().pin_memory() for x in (q, k, v))
    outp = torch.empty(qp.shape, dtype=torch.bfloat16).pin_memory()
    lsep = torch.empty(qp.shape[:3], dtype=torch.float32).pin_memory()
    cfg = fp.PipelineConfig()
    fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
        print(f"wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__" and not os.environ.get("FPB_CHUNK_KERNELS"):
    main()


def chunk_kernels(L=32768):
    """Device-resident kernel time of one e2e chunk (cq Q heads of one KV group)."""
    import math
    from tools.configs import timed
    q, k, v = workload.qwen3_30b_a3b(L, seed=1234, device="cuda")
    cfg = fp.PipelineConfig()
    grid = fp.make_block_grid(L, 128)
    for cq in (1, 2, 4, 8, 32):
        hk = 1 if cq < 32 else 4
        qs, ks, vs = q[:, :cq].contiguous(), k[:, :hk].contiguous(), v[:, :hk].contiguous()
        hold = {}

        def disc():
            hold["p"] = fp.discover_select(qs, ks, cfg)[0]
        td = timed(disc)
        ta = timed(lambda: fp.block_sparse_attention(qs, ks, vs, hold["p"], grid,
                                                     1 / math.sqrt(128)))
        print(f"chunk of {cq} Q heads: discover+select {td:.3f} ms, attention {ta:.3f} ms, "
              f"per head {(td + ta) / cq:.3f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__" and os.environ.get("FPB_CHUNK_KERNELS"):
    chunk_kernels()
