"""Parity at the BASELINE configurations' full sizes: the CUDA hot path (through the C ABI) against
the UNMODIFIED reference pipeline (oracle/_ref: discover -> max_threshold_mask -> compress_indices
-> block_sparse_attention, acceptance.cpp:357-360) on the same inputs.

BASELINE.json configs:
  C1  single head, 4K, d=128, fp32, planted vertical+slash          -> every row, whole pipeline
  C2  Qwen3-30B-A3B layer (32 Q / 4 KV), bf16, 32K                   -> 8 sampled Q heads, all rows
  C3  Llama-3.1-8B layer (32 Q / 8 KV), bf16, 64K                    -> 8 heads, sampled rows
  C4  Qwen3 shape, 128K, alpha sweep                                 -> 4 heads, masks at 3 alphas,
                                                                        attention on sampled rows
  C5  Qwen3 shape, 256K                                              -> 2 heads, sampled rows
The GPU always runs the whole layer (every head, every row: the plan-only hot path that bench.py
times — the two-pass select below 1024 key blocks, the prefilled fused epilogue from 1024); the
reference runs the sampled (z, h) slices with K/V of their KV head (GQA = per-Q-head reference
calls, SURVEY §7 hard part 5).  Bars: oracle/parity.py (north_star).  Each case prints its counts.
"""
import os

import numpy as np
import pytest
import torch

from oracle import parity

pytestmark = pytest.mark.gpu

THREADS = max(1, min(32, os.cpu_count() or 1))


def _sample_rows(M: int, n: int) -> np.ndarray:
    """Query blocks to attend on the CPU: first, last, and an even spread (long rows included)."""
    keep = np.zeros(M, bool)
    keep[np.unique(np.linspace(0, M - 1, n).round().astype(int))] = True
    keep[[0, M - 1]] = True
    return keep


def _run_case(fp, ref, q, k, v, cfg, heads, row_keep=None, alphas=None):
    """q/k/v: CUDA tensors of the whole layer.  Returns a summary dict (also printed)."""
    Z, Hq, L, d = q.shape
    Hkv = k.shape[1]
    B = cfg.block_size
    M = (L + B - 1) // B
    tau = cfg.resolved_scale(d)
    grid = fp.make_block_grid(L, B)
    # ---- GPU: the plan-only hot path + attention over the whole layer
    plan = fp.discover_select(q, k, cfg)[0]
    res = fp.block_sparse_attention(q, k, v, plan, grid, tau, out_dtype=torch.float32)
    torch.cuda.synchronize()
    hz = [(h // Hq, h % Hq) for h in heads]
    g_idx = np.stack([plan.indices[z, :, :, h].cpu().numpy() for z, h in hz])
    g_cnt = np.stack([plan.counts[z, :, h].cpu().numpy() for z, h in hz])
    keep = np.ones(M, bool) if row_keep is None else row_keep
    tok = torch.from_numpy(np.repeat(keep, B)[:L]).to(q.device)
    g_out = np.stack([res.out[z, h][tok].cpu().numpy() for z, h in hz])
    g_lse = np.stack([res.lse[z, h][tok].cpu().numpy() for z, h in hz])
    # ---- reference on the sampled slices (bf16 values upcast exactly)
    kvh = sorted({z * Hkv + h // (Hq // Hkv) for z, h in hz})
    qs = torch.stack([q[z, h] for z, h in hz]).float().cpu().numpy()[None]
    ks = torch.stack([k.reshape(Z * Hkv, L, d)[i] for i in kvh]).float().cpu().numpy()[None]
    vs = torch.stack([v.reshape(Z * Hkv, L, d)[i] for i in kvh]).float().cpu().numpy()[None]
    # re-index: sampled slice s reads reference KV slice kvh.index(...) -> run one call per slice
    # through a (1, n, L, d) Q batch whose KV heads are listed per slice (Hq = Hkv = n)
    ks_s = np.stack([ks[0, kvh.index(z * Hkv + h // (Hq // Hkv))] for z, h in hz])[None]
    vs_s = np.stack([vs[0, kvh.index(z * Hkv + h // (Hq // Hkv))] for z, h in hz])[None]
    r = ref.pipeline_detail(qs, ks_s, vs_s, B, cfg.alpha, cfg.sink_tokens, cfg.window_tokens,
                            tau, cfg.epsilon, list(range(len(hz))), THREADS,
                            row_keep=None if row_keep is None else row_keep)
    pp = parity.compare_plans(g_idx, g_cnt, r["idx"], r["counts"], r["score"], cfg.alpha)
    rows_ok = pp["same_row"] & keep[None, :]
    r_out = np.stack([r["out"][s][np.repeat(keep, B)[:L]] for s in range(len(hz))])
    r_lse = np.stack([r["lse"][s][np.repeat(keep, B)[:L]] for s in range(len(hz))])
    po = parity.compare_outputs(g_out, g_lse, r_out, r_lse, rows_ok[:, keep], B)
    summary = {k2: v2 for k2, v2 in pp.items() if k2 != "same_row"}
    summary.update(po)
    summary["ref_secs"] = round(r["secs"], 2)
    print(f"L={L} Hq={Hq} Hkv={Hkv} heads={heads}: {summary}")
    assert pp["mismatch_outside_band"] == 0, summary
    assert pp["rows_differ_without_near"] == 0, summary
    assert po["tokens"] > 0
    assert po["out_max"] <= parity.OUT_MAX_ABS and po["out_mean"] <= parity.OUT_MEAN_ABS, summary
    assert po["lse_max"] <= parity.OUT_MAX_ABS and po["lse_mean"] <= parity.OUT_MEAN_ABS, summary
    # visits: the GPU counts of the sampled heads equal the reference's wherever rows agree
    for a in alphas or ():
        c2 = fp.PipelineConfig(alpha=a, sink_tokens=cfg.sink_tokens,
                               window_tokens=cfg.window_tokens)
        p2 = fp.discover_select(q, k, c2)[0]
        gi2 = np.stack([p2.indices[z, :, :, h].cpu().numpy() for z, h in hz])
        gc2 = np.stack([p2.counts[z, :, h].cpu().numpy() for z, h in hz])
        sc = r["score"]
        masks = [ref.max_threshold_mask(sc[s][None, None], B, a, cfg.sink_tokens,
                                        cfg.window_tokens)[0] for s in range(len(hz))]
        ri, rc = zip(*(ref.compress_indices(m) for m in masks))
        ri = np.stack([x[0, :, :, 0] for x in ri])
        rc = np.stack([x[0, :, 0] for x in rc])
        pa = parity.compare_plans(gi2, gc2, ri, rc, sc, a)
        dens = float(gc2.sum()) / (len(hz) * M * (M + 1) / 2)
        print(f"  alpha={a}: density {dens:.4f} "
              f"{ {k2: v2 for k2, v2 in pa.items() if k2 != 'same_row'} }")
        assert pa["mismatch_outside_band"] == 0 and pa["rows_differ_without_near"] == 0
    return summary


def test_c1_single_head_4k_fp32(fp, ref):
    """C1 exactly: one head, L = 4096, d = 128, fp32 inputs, whole pipeline on every row."""
    q, k, v = fp.workload.composite(101, 1, 1, 1, 4096, dtype=torch.float32)
    q, k, v = (x.cuda() for x in (q, k, v))
    _run_case(fp, ref, q, k, v, fp.PipelineConfig(), [0])


def test_c2_qwen3_32k(fp, ref):
    """C2: Qwen3-30B-A3B layer at 32K (the bench workload and seed), 8 Q heads over all 4 KV
    groups, every row."""
    q, k, v = fp.workload.composite(1234, 1, 32, 4, 32768)  # bench.py make_inputs(seq 0)
    q, k, v = (x.cuda() for x in (q, k, v))
    heads = [0, 8, 16, 24, 5, 13, 22, 31]
    _run_case(fp, ref, q, k, v, fp.PipelineConfig(alpha=0.12), heads)


def test_c3_llama_64k(fp, ref):
    """C3: Llama-3.1-8B layer (32 Q / 8 KV) at 64K, one Q head per KV group, 40 sampled rows."""
    L = 65536
    q, k, v = fp.workload.llama31_8b(L, seed=5, device="cuda")
    heads = [h * 4 + (h % 4) for h in range(8)]
    _run_case(fp, ref, q, k, v, fp.PipelineConfig(alpha=0.12), heads,
              row_keep=_sample_rows(L // 128, 40))


def test_c4_qwen3_128k_alpha_sweep(fp, ref):
    """C4: Qwen3 shape at 128K (M = 1024: the prefilled long-row epilogue), one Q head per KV
    group; masks at alpha 0.05 / 0.12 / 0.3 against the reference selector on the reference's own
    score map; attention on 16 sampled rows."""
    L = 131072
    q, k, v = fp.workload.qwen3_30b_a3b(L, seed=9, device="cuda")
    _run_case(fp, ref, q, k, v, fp.PipelineConfig(alpha=0.12), [3, 9, 18, 28],
              row_keep=_sample_rows(L // 128, 16), alphas=(0.05, 0.3))


def test_c5_qwen3_256k(fp, ref):
    """C5: Qwen3 shape at 256K (M = 2048), two Q heads of different KV groups, 8 sampled rows."""
    L = 262144
    q, k, v = fp.workload.qwen3_30b_a3b(L, seed=13, device="cuda")
    _run_case(fp, ref, q, k, v, fp.PipelineConfig(alpha=0.12), [6, 25],
              row_keep=_sample_rows(L // 128, 8))
