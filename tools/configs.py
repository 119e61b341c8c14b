#!/usr/bin/env python
"""Run every BASELINE.json config on one B200 and print one JSON line per measurement.

  C1  single head, 4K, d 128, fp32 synthetic Q/K/V (CPU reference runs in full beside it)
  C2  Qwen3-30B-A3B layer (32 Q / 4 KV), bf16, 32K                      (== bench.py default)
  C3  Llama-3.1-8B layer (32 Q / 8 KV), bf16, 64K; plus one rank's KV-group shard at G=2/4/8
  C4  Qwen3 shape at 128K, alpha sweep: density, visits, error vs the dense kernel, stage ms
  C5  Qwen3 shape at 256K: pool / discover+select / attention breakdown; one rank's 1/8 shard

usage: python tools/configs.py [--only C1,C4] [--out profiles/r1_configs.jsonl]
Multi-GPU numbers are NOT produced here (one GPU per box); shard rows time one rank's share.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import shard, workload  # noqa: E402

D = 128


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def dense_flops(Z, H, L):
    return 4.0 * D * Z * H * L * (L + 1) / 2.0


def stage_times(q, k, v, cfg, out_dtype=torch.bfloat16):
    """Device time of each stage, replayed from CUDA graphs (PrefillRunner): no host work in
    the timed region.  discover+select includes its key pooling."""
    L = q.shape[2]
    grid = fp.make_block_grid(L, 128)
    t_pool = timed(lambda: fp.pool_keys(k, grid))
    r = fp.PrefillRunner(q, k, v, cfg, out_dtype=out_dtype).capture()
    t_disc = timed(r.replay_discover)
    t_attn = timed(r.replay_attend)
    r.check()
    plan = fp.SparseBlockPlan(r.idx.clone(), r.counts.clone())
    visits = int(plan.counts.to(torch.int64).sum())
    M = grid.num_query_blocks
    dens = visits / (q.shape[0] * q.shape[1] * M * (M + 1) / 2)
    return dict(pool_ms=t_pool, discover_select_ms=t_disc, attention_ms=t_attn,
                step_ms=t_disc + t_attn, visits=visits, density=dens), plan


def c1(emit):
    from oracle import Oracle, available
    L = 4096
    q, k, v = workload.composite(1, 1, 1, 1, L, dtype=torch.float32)
    cfg = fp.PipelineConfig()
    qd, kd, vd = (x.cuda() for x in (q, k, v))
    st, plan = stage_times(qd, kd, vd, cfg, out_dtype=torch.float32)
    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    t0 = time.time()
    secs, ro, rl, rvis = o.pipeline(q.numpy(), k.numpy(), v.numpy(), 128, cfg.alpha, 256, 512,
                                    cfg.resolved_scale(D), 1e-10, [0], 1)
    res = fp.prefill(qd, kd, vd, cfg, out_dtype=torch.float32)[0]
    err = (res.out[0, 0].cpu() - torch.from_numpy(ro[0])).abs()
    lerr = (res.lse[0, 0].cpu() - torch.from_numpy(rl[0])).abs()
    emit(dict(config="C1 single head 4K fp32", **st, cpu_reference_ms=secs * 1e3,
              cpu_kind=kind, cpu_visits=rvis, out_max_abs=float(err.max()),
              out_mean_abs=float(err.mean()), lse_max_abs=float(lerr.max()),
              speedup_vs_cpu=secs * 1e3 / st["step_ms"]))


def c2(emit):
    q, k, v = (x.cuda() for x in workload.qwen3_30b_a3b(32768, seed=1234))
    st, _ = stage_times(q, k, v, fp.PipelineConfig())
    t_dense = timed(lambda: fp.dense_attention(q, k, v, 1 / math.sqrt(D)), reps=3)
    emit(dict(config="C2 Qwen3 32K bf16", **st, dense_ms=t_dense,
              speedup_vs_dense=t_dense / st["step_ms"],
              eff_tflops=dense_flops(1, 32, 32768) / st["step_ms"] / 1e9))


def c3(emit):
    L = 65536
    q, k, v = workload.llama31_8b(L, seed=7, device="cuda")
    st, _ = stage_times(q, k, v, fp.PipelineConfig(alpha=0.18))
    t_dense = timed(lambda: fp.dense_attention(q, k, v, 1 / math.sqrt(D)), reps=2, warm=1)
    emit(dict(config="C3 Llama-3.1-8B 64K bf16 alpha=0.18, 1 GPU", alpha=0.18, **st, dense_ms=t_dense,
              speedup_vs_dense=t_dense / st["step_ms"],
              eff_tflops=dense_flops(1, 32, L) / st["step_ms"] / 1e9))
    for G in (2, 4, 8):
        s = shard.kv_group_shard(32, 8, G, 0)
        ql, kl, vl = shard.local_slices(q, k, v, s)
        st2, _ = stage_times(ql, kl, vl, fp.PipelineConfig(alpha=0.18))
        emit(dict(config=f"C3 Llama 64K: one rank's KV-group shard at G={G} "
                         f"({s.hq} Q / {s.hkv} KV heads), timed alone on 1 GPU", alpha=0.18, **st2,
                  eff_tflops_per_gpu=dense_flops(1, s.hq, L) / st2["step_ms"] / 1e9))


def c4(emit):
    L = 131072
    q, k, v = (x for x in workload.composite(11, 1, 32, 4, L, device="cuda"))
    grid = fp.make_block_grid(L, 128)
    tau = 1 / math.sqrt(D)
    dense = fp.dense_attention(q, k, v, tau, out_dtype=torch.float32)
    t_dense = timed(lambda: fp.dense_attention(q, k, v, tau), reps=2, warm=1)
    for a in (0.0, 0.02, 0.05, 0.08, 0.12, 0.18, 0.3, 0.5, 1.0):
        cfg = fp.PipelineConfig(alpha=a)
        st, plan = stage_times(q, k, v, cfg)
        res = fp.block_sparse_attention(q, k, v, plan, grid, tau, out_dtype=torch.float32)
        err = (res.out - dense.out).abs()
        emit(dict(config=f"C4 Qwen3 128K alpha sweep", alpha=a, **st, dense_ms=t_dense,
                  speedup_vs_dense=t_dense / st["step_ms"],
                  err_max_abs=float(err.max()), err_mean_abs=float(err.mean()),
                  eff_tflops=dense_flops(1, 32, L) / st["step_ms"] / 1e9))
        del res, err


def c5(emit):
    L = 262144
    q, k, v = workload.composite(5, 1, 32, 4, L, device="cuda")
    st, _ = stage_times(q, k, v, fp.PipelineConfig())
    emit(dict(config="C5 Qwen3 256K bf16, 1 GPU (all 32 heads)", **st,
              eff_tflops=dense_flops(1, 32, L) / st["step_ms"] / 1e9))
    s = shard.kv_group_shard(32, 4, 8, 0)
    ql, kl, vl = shard.local_slices(q, k, v, s)
    st2, _ = stage_times(ql, kl, vl, fp.PipelineConfig())
    emit(dict(config="C5 Qwen3 256K: one rank's 1/8 shard (4 Q / 1 KV heads), timed alone",
              **st2, eff_tflops_per_gpu=dense_flops(1, s.hq, L) / st2["step_ms"] / 1e9))


def to_markdown(path):
    """Render a configs .jsonl as the markdown table committed under profiles/."""
    rows = [json.loads(x) for x in open(path)]
    out = ["# BASELINE configs on one B200 (tools/configs.py; CUDA events, median of 5; stage "
           "times are CUDA-graph replays; bf16 unless noted)", "",
           "| config | alpha | density | visits | pool ms | discover+select ms | attention ms | "
           "step ms | dense K5 ms | speedup vs dense | err max / mean vs dense |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        err = (f"{r['err_max_abs']:.3g} / {r['err_mean_abs']:.3g}" if "err_max_abs" in r else "-")
        out.append(
            f"| {r['config']} | {r.get('alpha', 0.12)} | {r['density']:.3f} | {r['visits']} | "
            f"{r['pool_ms']:.3f} | {r['discover_select_ms']:.3f} | {r['attention_ms']:.3f} | "
            f"{r['step_ms']:.3f} | {r['dense_ms']:.2f} | {r['speedup_vs_dense']:.2f} | {err} |"
            if "dense_ms" in r else
            f"| {r['config']} | {r.get('alpha', 0.12)} | {r['density']:.3f} | {r['visits']} | "
            f"{r['pool_ms']:.3f} | {r['discover_select_ms']:.3f} | {r['attention_ms']:.3f} | "
            f"{r['step_ms']:.3f} | - | - | {err} |")
    c1 = [r for r in rows if r["config"].startswith("C1")]
    if c1:
        r = c1[0]
        out += ["", f"C1 (fp32, 4K, 1 head): GPU step {r['step_ms']:.3f} ms vs the reference CPU "
                    f"pipeline {r['cpu_reference_ms']:.1f} ms (1 thread, oracle/{r['cpu_kind']}) = "
                    f"{r['speedup_vs_cpu']:.0f}x; same plan visits ({r['visits']} = "
                    f"{r['cpu_visits']}); out max-abs {r['out_max_abs']:.2e}, mean-abs "
                    f"{r['out_mean_abs']:.2e}, lse max-abs {r['lse_max_abs']:.2e}."]
    out += ["Shard rows time ONE rank's KV-group shard alone on one GPU (the box has one GPU); "
            "they are not multi-GPU measurements (profiles/r1_lsweep.md has every rank's share "
            "and the row-sharded partition)."]
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--out", default="")
    ap.add_argument("--markdown", default="", help="render this .jsonl and exit")
    args = ap.parse_args()
    if args.markdown:
        print(to_markdown(args.markdown), end="")
        return
    f = open(args.out, "a") if args.out else None

    def emit(d):
        line = json.dumps(d)
        print(line, flush=True)
        if f:
            f.write(line + "\n")
            f.flush()
    for name in args.only.split(","):
        {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[name](emit)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
