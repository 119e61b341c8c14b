#!/usr/bin/env python
"""Sparse-prefill latency across sequence lengths at the Qwen3-30B-A3B layer shape (32 Q / 4 KV
heads, d 128, bf16, alpha 0.12), one B200, plus one KV-group shard per rank at G = 2/4/8.

Per length: pool / discover+select / sparse attention / dense K5 ms (CUDA events, median), density,
effective TFLOP/s (dense-causal-equivalent), the attention kernel's algorithmic
TFLOP/s and its fraction of the measured sustained bf16 peak, discovery GB/s against HBM.
Shard rows: every rank's share (kv_group_shard) timed alone on this GPU; the G-GPU step is the max
over ranks (no data-path collective; the O/LSE all-gather bytes per rank are listed, not timed:
the pool gives one GPU per box).

usage: python tools/lsweep.py [--Ls 4096,...] [--out profiles/r1_lsweep.jsonl]
       python tools/lsweep.py --markdown profiles/r1_lsweep.jsonl > profiles/r1_lsweep.md
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
from paper_2603_06199_b200 import shard, workload  # noqa: E402
from tools.configs import timed  # noqa: E402

D = 128
HQ, HKV = 32, 4


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except OSError:
        p = {}

    def pick(*keys, default):
        for k in keys:
            if isinstance(p.get(k), (int, float)):
                return float(p[k])
        return default
    # burst bf16 peak: each stage is timed as a short burst at full clock (bench.py does the same)
    return (pick("hbm_gbs", "hbm_gbps", default=6553.3),
            pick("bf16_tflops", "bf16_dense_tflops", default=1643.8))


def plan_flops(plan):
    c = int(plan.counts.to(torch.int64).sum())
    ndiag = plan.counts.numel()
    return (c - ndiag) * 4.0 * D * 128 * 128 + ndiag * 4.0 * D * 128 * 129 / 2, c


def stage(q, k, v, cfg, grid, tau, reps, rows=None):
    """Device time of the two stages, each replayed from a CUDA graph (PrefillRunner)."""
    r = fp.PrefillRunner(q, k, v, cfg, rows=rows).capture()
    t_disc = timed(r.replay_discover, reps=reps, warm=1)
    t_attn = timed(r.replay_attend, reps=reps, warm=1)
    r.check()
    plan = r.plan
    if rows is not None:
        return t_disc, t_attn, 0.0, 0
    fl, visits = plan_flops(plan)
    return t_disc, t_attn, fl, visits


def _kl(L):
    return f"{L // 1024}K"


def markdown(path):
    """Render a sweep .jsonl as the tables in profiles/r1_lsweep.md."""
    recs = [json.loads(x) for x in open(path) if x.strip()]
    _, tc = peaks()
    one = [r for r in recs if r["G"] == 1]
    print("# Sparse-prefill latency vs sequence length — Qwen3-30B-A3B layer (32 Q / 4 KV heads, "
          f"d 128), bf16, alpha {one[0]['alpha'] if one else 0.12}\n")
    print("`tools/lsweep.py` on one B200: each stage replayed from a CUDA graph (`PrefillRunner`), "
          "CUDA events, median of 3-5; inputs resident in HBM; synthetic vertical+slash composite, "
          "seed 5.")
    print("Attention fraction = plan FLOPs (4dB^2 per off-diagonal visit, 4dB(B+1)/2 per diagonal "
          f"visit) / kernel time / {tc} TFLOP/s")
    print("(MEASURED_PEAKS.json burst bf16, recomputed from the recorded algorithmic TFLOP/s). "
          "Discovery bytes = Q + K read + idx (M x N) + counts written (SURVEY §8d).\n")
    print("| L | density | pool ms | discover+select ms | sparse attn ms | step ms | dense K5 ms | "
          "speedup vs dense | eff. TFLOP/s (dense-equiv) | attn alg. TFLOP/s | attn frac | "
          "discovery GB/s | disc frac of HBM |")
    print("|" + "---|" * 13)
    for r in one:
        dense = f"{r['dense_ms']:.2f}" if "dense_ms" in r else "-"
        sp = f"{r['speedup_vs_dense']:.2f}" if "speedup_vs_dense" in r else "-"
        print(f"| {_kl(r['L'])} | {r['density']:.3f} | {r['pool_ms']:.3f} | "
              f"{r['discover_select_ms']:.3f} | {r['attention_ms']:.3f} | {r['step_ms']:.3f} | "
              f"{dense} | {sp} | {r['eff_tflops']:.0f} | {r['attn_alg_tflops']:.0f} | "
              f"{r['attn_alg_tflops'] / tc:.3f} | {r['disc_gbps']:.0f} | {r['disc_frac']:.3f} |")
    print("\n## 2 / 4 / 8 GPUs: every rank's share timed alone on this GPU (the pool gives one GPU "
          "per box)\n")
    print("Step = max over ranks (no data-path collective). `kv_group`: the north_star partition "
          "(rank owns KV heads; Qwen3 at 8 ranks splits each group's 8 Q heads 4+4).")
    print("`kv_zigzag`: one KV head per rank as in kv_group, but the G/Hkv ranks of a group "
          "each take all of its Q heads and split the query blocks in zigzag chunks (G = 8 only; "
          "identical to kv_group for G <= Hkv). `kv_weighted`: the same with ranks per KV group "
          "by the layer plan's visits per group (`shard.kv_group_ranks`).")
    print("`rows`: rank r owns query blocks r, r+G, ... of every head (`fpb_*_rows`), K/V "
          "replicated. `zigzag`: rank r owns contiguous chunks r and 2G-1-r of 2G chunks "
          "(`fpb_*_zigzag`), K/V replicated. The O+LSE all-gather after the kernels is not timed "
          "(bytes listed; ~2 ms at 256K/8 ranks at ~900 GB/s).\n")
    print("| L | G | partition | step ms (max over ranks) | per-rank step ms | job eff. TFLOP/s | "
          "all-gather bytes per rank |")
    print("|" + "---|" * 7)
    for r in recs:
        if r["G"] == 1:
            continue
        ranks = ", ".join(f"{x:.2f}" for x in r["rank_step_ms"])
        print(f"| {_kl(r['L'])} | {r['G']} | {r['partition']} | "
              f"{r['step_ms_max_over_ranks']:.3f} | {ranks} | {r['eff_tflops_job']:.0f} | "
              f"{r['gather_bytes_per_rank'] / 2**20:.0f} MiB |")


def main():
    if len(sys.argv) == 3 and sys.argv[1] == "--markdown":
        markdown(sys.argv[2])
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--Ls", default="4096,8192,16384,32768,65536,131072,262144")
    ap.add_argument("--alpha", type=float, default=0.12)
    ap.add_argument("--out", default="")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--Gs", default="2,4,8")
    ap.add_argument("--parts", default="kv_group,kv_zigzag,kv_weighted,rows,zigzag")
    args = ap.parse_args()
    hbm, tc = peaks()
    out = open(args.out, "a") if args.out else None
    cfg = fp.PipelineConfig(alpha=args.alpha)
    tau = cfg.resolved_scale(D)
    for L in (int(x) for x in args.Ls.split(",")):
        torch.cuda.empty_cache()
        q, k, v = workload.composite(5, 1, HQ, HKV, L, device="cuda")
        grid = fp.make_block_grid(L, 128)
        M = grid.num_query_blocks
        reps = 5 if L <= 65536 else 3
        t_pool = timed(lambda: fp.pool_keys(k, grid), reps=reps, warm=1)
        t_disc, t_attn, fl, visits = stage(q, k, v, cfg, grid, tau, reps)
        dense_fl = 4.0 * D * HQ * L * (L + 1) / 2
        disc_bytes = HQ * L * D * 2 + HKV * L * D * 2 + HQ * M * M * 4 + HQ * M * 4
        rec = dict(L=L, alpha=args.alpha, G=1, density=visits / (HQ * M * (M + 1) / 2),
                   visits=visits, pool_ms=t_pool, discover_select_ms=t_disc,
                   attention_ms=t_attn, step_ms=t_disc + t_attn,
                   eff_tflops=dense_fl / (t_disc + t_attn) / 1e9,
                   attn_alg_tflops=fl / t_attn / 1e9, attn_frac=fl / t_attn / 1e9 / tc,
                   disc_gbps=disc_bytes / t_disc / 1e6, disc_frac=disc_bytes / t_disc / 1e6 / hbm)
        if not args.no_dense:
            t_dense = timed(lambda: fp.dense_attention(q, k, v, tau), reps=2, warm=1)
            rec.update(dense_ms=t_dense, speedup_vs_dense=t_dense / (t_disc + t_attn),
                       dense_tflops=dense_fl / t_dense / 1e9)
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
        # per-KV-group block visits of the whole layer (the kv_weighted partition's calibration)
        cnt = fp.discover_select(q, k, cfg)[0].counts.sum(dim=(0, 1)).double()
        gq = HQ // HKV
        kvw = [float(cnt[i * gq:(i + 1) * gq].sum()) for i in range(HKV)]
        for G in (int(x) for x in args.Gs.split(",")):
            for part in args.parts.split(","):
                if part in ("kv_zigzag", "kv_weighted") and G <= HKV:
                    continue  # identical to kv_group
                per_rank = []
                for rank in range(G):
                    if part in ("kv_zigzag", "kv_weighted"):
                        s, rows = shard.kv_zigzag_shard(HQ, HKV, G, rank,
                                                        kvw if part == "kv_weighted" else None)
                        ql, kl, vl = (x.contiguous() for x in shard.local_slices(q, k, v, s))
                        td, ta, _, vis = stage(ql, kl, vl, cfg, grid, tau, reps, rows=rows)
                    elif part == "kv_group":
                        s = shard.kv_group_shard(HQ, HKV, G, rank)
                        ql, kl, vl = (x.contiguous() for x in shard.local_slices(q, k, v, s))
                        td, ta, _, vis = stage(ql, kl, vl, cfg, grid, tau, reps)
                    else:
                        rows = (shard.row_shard(G, rank) if part == "rows"
                                else shard.zigzag_shard(G, rank))
                        td, ta, _, vis = stage(q, k, v, cfg, grid, tau, reps, rows=rows)
                    per_rank.append((td + ta, td, ta, vis))
                worst = max(per_rank)
                gather = (G - 1) / G * HQ * L * (D * 2 + 4)  # bf16 O + fp32 LSE received per rank
                rec = dict(L=L, alpha=args.alpha, G=G, partition=part,
                           step_ms_max_over_ranks=worst[0],
                           discover_select_ms=worst[1], attention_ms=worst[2],
                           rank_step_ms=[round(x[0], 4) for x in per_rank],
                           eff_tflops_job=dense_fl / worst[0] / 1e9,
                           gather_bytes_per_rank=int(gather))
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
        del q, k, v


if __name__ == "__main__":
    main()
