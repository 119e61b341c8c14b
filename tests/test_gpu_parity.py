"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle on identical inputs.

Bars (north_star / SURVEY §8c):
  * pooled keys, threshold mask, compaction: bit-exact given identical inputs;
  * discovery mask / idx / counts: bit-exact except blocks whose reference score lies within
    MASK_EPS * thresh of the threshold (counted and reported);
  * attention out: max-abs <= 2e-2 and mean-abs <= 1e-3 against the reference's fp32 result on the
    same plan; lse compared in base 2 with the same bars.
"""
import numpy as np
import pytest
import torch

from tests._util import (MASK_EPS, OUT_MAX_ABS, OUT_MEAN_ABS, bf16_round, compare_masks,
                         composite_np, err, rows_with_near)

pytestmark = pytest.mark.gpu


def _cuda(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _np(t):
    return t.detach().float().cpu().numpy() if t.dtype != torch.uint8 and t.dtype != torch.int32 \
        else t.cpu().numpy()


def _planted(port, kind, a, b, L, H=2, seed=3, strength=2.5):
    q, k, v, _ = port.generate_planted(kind, strength, a, b, 0.5, seed, 1, H, L, 128, 128)
    return bf16_round(q), bf16_round(k), bf16_round(v)


# --------------------------------------------------------------------------- pooling (K1)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("L", [128, 1000, 2048])
def test_pool_keys_bitexact(fp, port, dtype, L):
    rng = np.random.default_rng(L)
    k = rng.normal(0, 1, (2, 3, L, 128)).astype(np.float32)
    if dtype == torch.bfloat16:
        k = bf16_round(k)
    got = _np(fp.pool_keys(_cuda(k, dtype), fp.make_block_grid(L, 128)).data)
    want = port.pool_keys(k, 128)
    assert np.array_equal(got, want)


# --------------------------------------------------------------------------- discovery (K2)
@pytest.mark.parametrize("case", [(0, 3, 0, 2048), (1, 300, 0, 2048), (1, 777, 0, 1000),
                                  (2, 9, 4, 1536), (3, 1500, 0, 4096)])
def test_discover_maps(fp, port, case):
    kind, a, b, L = case
    q, k, v = _planted(port, kind, a, b, L)
    tau = float(port.scale(128))
    en, lm, sc = port.discover(q, k, 128, tau)
    m = fp.discover(_cuda(q), _cuda(k), fp.make_block_grid(L, 128), tau)
    gen, glm, gsc = _np(m.energy), _np(m.local_max), _np(m.score)
    M = sc.shape[2]
    tri = np.tril(np.ones((M, M), bool))[None, None]
    # non-causal sentinels are exact (discovery.hpp:84, 124)
    assert np.all(gen[:, :, ~tri[0, 0]] == 0) and np.all(gsc[:, :, ~tri[0, 0]] == 0)
    assert np.all(glm[:, :, ~tri[0, 0]] == np.finfo(np.float32).min)
    # causal entries: local max (base-2 logit units) and scores close to the fp32 reference
    dl = np.abs(glm - lm)[np.broadcast_to(tri, lm.shape)]
    assert dl.max() <= 2e-4 * max(1.0, np.abs(lm[np.broadcast_to(tri, lm.shape)]).max())
    # scores: relative 5e-5 (SURVEY §7 targets the reference's own 1e-5 energy bar,
    # test_discovery.cpp:114-116; k̄ enters as a 16-significant-bit hi+lo split and exp2 is
    # ex2.approx, so a few ulps more are allowed, far inside the 1e-4 mask band)
    rs = np.abs(gsc - sc) / np.maximum(sc, 1e-30)
    big = np.broadcast_to(tri, sc.shape) & (sc > 1e-6)
    print(f"score rel err max {rs[big].max():.2e} mean {rs[big].mean():.2e}")
    assert rs[big].max() <= 5e-5, rs[big].max()


@pytest.mark.parametrize("shape", [(1, 2, 2, 2048), (2, 6, 3, 1000), (1, 4, 1, 300)])
def test_in_kernel_pooling_bit_identical(fp, port, shape):
    """bf16 discovery pools K inside the discovery kernel (claimed blocks, per-chunk release /
    acquire counters); the result must equal the two-launch path — pool_keys (bit-exact against
    the oracle) then approx_block_scores on that k̄ — bit for bit, ragged last block and GQA
    included."""
    Z, Hq, Hkv, L = shape
    q, k, _ = (bf16_round(x) for x in composite_np(7 + L, Z, Hq, Hkv, L))
    grid = fp.make_block_grid(L, 128)
    tau = float(port.scale(128))
    pk = fp.pool_keys(_cuda(k), grid)
    assert np.array_equal(_np(pk.data), port.pool_keys(k, 128))
    two = fp.approx_block_scores(_cuda(q), pk, grid, tau)
    one = fp.discover(_cuda(q), _cuda(k), grid, tau)
    assert np.array_equal(_np(one.energy), _np(two.energy))
    assert np.array_equal(_np(one.local_max), _np(two.local_max))


def test_discovery_on_concurrent_streams(fp):
    """Two streams run persistent discovery launches (one CTA per SM each, in-kernel pooling with
    cross-CTA counters) at the same time, so each launch gets only part of the SMs; claims are
    dynamic, so neither may wait on a pooling unit held by a CTA that is not running.  Plans equal
    the single-stream ones."""
    L = 8192
    q, k, _ = (bf16_round(x) for x in composite_np(11, 1, 32, 4, L))
    q2 = np.ascontiguousarray(q[:, ::-1])
    cfg = fp.PipelineConfig()
    ins = [(_cuda(q), _cuda(k)), (_cuda(q2), _cuda(k))]
    ref = [fp.discover_select(a, b, cfg)[0] for a, b in ins]
    ref = [(_np(p.indices), _np(p.counts)) for p in ref]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    outs = [[], []]
    for _ in range(6):
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                outs[i].append(fp.discover_select(*ins[i], cfg)[0])
    torch.cuda.synchronize()
    for i in range(2):
        for p in outs[i]:
            assert np.array_equal(_np(p.indices), ref[i][0])
            assert np.array_equal(_np(p.counts), ref[i][1])


@pytest.mark.parametrize("alpha", [0.0, 0.05, 0.12, 0.5, 1.0])
def test_threshold_and_compress_bitexact(fp, port, alpha):
    q, k, _ = _planted(port, 1, 300, 0, 4096, H=3)
    tau = float(port.scale(128))
    _, _, sc = port.discover(q, k, 128, tau)
    cfg = fp.PipelineConfig(alpha=alpha)
    st = fp.SelectionStats()
    gm = fp.max_threshold_mask(_cuda(sc, torch.float32), cfg, st)
    mask, cmp = port.max_threshold_mask(sc, 128, alpha, 256, 512)
    assert np.array_equal(_np(gm.active), mask)
    assert st.score_comparisons == cmp
    plan = fp.compress_indices(gm)
    idx, counts = port.compress_indices(mask)
    assert np.array_equal(_np(plan.indices), idx) and np.array_equal(_np(plan.counts), counts)
    assert fp.visit_count(plan) == port.visit_count(counts)


def test_compress_arbitrary_mask(fp, port):
    rng = np.random.default_rng(5)
    mask = (rng.random((2, 17, 17, 5)) < 0.3).astype(np.uint8)  # includes j > i entries
    plan = fp.compress_indices(fp.ActiveMask(_cuda(mask, torch.uint8)))
    idx, counts = port.compress_indices(mask)
    assert np.array_equal(_np(plan.indices), idx) and np.array_equal(_np(plan.counts), counts)


@pytest.mark.parametrize("shape", [(1, 2, 2, 2048), (1, 4, 2, 3000), (2, 2, 1, 1024),
                                   (1, 8, 2, 4096)])
@pytest.mark.parametrize("alpha", [0.0, 0.05, 0.12, 0.3])
@pytest.mark.parametrize("with_maps", [True, False])
def test_fused_discover_select(fp, port, shape, alpha, with_maps):
    """with_maps=False is the plan-only hot path (log-domain threshold, two barrier rounds);
    with_maps=True also writes the score map (linear-domain threshold, three rounds)."""
    Z, Hq, Hkv, L = shape
    q, k, v = composite_np(11 + L, Z, Hq, Hkv, L)
    q, k = bf16_round(q), bf16_round(k)
    tau = float(port.scale(128))
    _, _, sc = port.discover(q, k, 128, tau)
    mask, _ = port.max_threshold_mask(sc, 128, alpha, 256, 512)
    idx, counts = port.compress_indices(mask)
    cfg = fp.PipelineConfig(alpha=alpha)
    plan, smap, gmask = fp.discover_select(_cuda(q), _cuda(k), cfg, want_score=with_maps,
                                           want_mask=True)
    bad, near, flipped = compare_masks(_np(gmask.active), mask, sc, alpha)
    print(f"shape={shape} alpha={alpha} maps={with_maps}: near-threshold blocks={near} "
          f"flipped={flipped}")
    assert bad == 0
    ok_rows = ~rows_with_near(sc, alpha)
    gi, gc = _np(plan.indices), _np(plan.counts)
    assert np.array_equal(gc[ok_rows], counts[ok_rows])
    assert np.array_equal(gi.transpose(0, 1, 3, 2)[ok_rows], idx.transpose(0, 1, 3, 2)[ok_rows])


@pytest.mark.parametrize("shape", [(1, 40, 8, 1000), (1, 64, 8, 700), (2, 6, 3, 1300),
                                   (1, 1, 1, 2000), (1, 12, 4, 777)])
def test_plan_only_two_pass_head_counts(fp, port, shape):
    """Plan-only calls below 1024 key blocks run the two-pass path (discovery writes the (m, S)
    triangle, select_rows assembles each head-last plan row slab).  Head counts that are not a
    power of two, exceed one 32-head slab, or are 1 exercise the slab chunking and the scalar
    copy-out; the plan must equal the reference outside the epsilon band (selection.hpp:63-92,
    176-192)."""
    Z, Hq, Hkv, L = shape
    q, k, _ = composite_np(7 + L, Z, Hq, Hkv, L)
    q, k = bf16_round(q), bf16_round(k)
    tau = float(port.scale(128))
    kk = np.repeat(k, Hq // Hkv, axis=1)
    _, _, sc = port.discover(q, kk, 128, tau)
    mask, _ = port.max_threshold_mask(sc, 128, 0.12, 256, 512)
    idx, counts = port.compress_indices(mask)
    plan = fp.discover_select(_cuda(q), _cuda(k), fp.PipelineConfig(alpha=0.12))[0]
    gi, gc = _np(plan.indices), _np(plan.counts)
    M = gc.shape[1]
    zz, ii, ss, hh = np.meshgrid(np.arange(Z), np.arange(M), np.arange(M), np.arange(Hq),
                                 indexing="ij")
    live = ss < gc[:, :, None, :]
    assert bool((gi[~live] == M).all())
    gmask = np.zeros((Z, M, M + 1, Hq), bool)
    gmask[zz[live], ii[live], gi[live], hh[live]] = True
    bad, near, flipped = compare_masks(gmask[:, :, :M], mask, sc, 0.12)
    assert bad == 0, (bad, near, flipped)
    ok_rows = ~rows_with_near(sc, 0.12)
    assert np.array_equal(gc[ok_rows], counts[ok_rows])
    assert np.array_equal(gi.transpose(0, 1, 3, 2)[ok_rows], idx.transpose(0, 1, 3, 2)[ok_rows])


def test_fused_discover_select_global_rows(fp, port, monkeypatch):
    """The long-sequence variant (per-key-block rows in a global scratch instead of shared memory,
    taken automatically beyond ~270K tokens) forced at a size the oracle finishes quickly."""
    monkeypatch.setenv("FPB_DISC_FORCE_SCRATCH", "1")
    Z, Hq, Hkv, L = 1, 4, 2, 3000
    q, k, v = composite_np(23, Z, Hq, Hkv, L)
    q, k = bf16_round(q), bf16_round(k)
    tau = float(port.scale(128))
    _, _, sc = port.discover(q, k, 128, tau)
    mask, _ = port.max_threshold_mask(sc, 128, 0.12, 256, 512)
    idx, counts = port.compress_indices(mask)
    plan, smap, gmask = fp.discover_select(_cuda(q), _cuda(k), fp.PipelineConfig(alpha=0.12),
                                           want_score=True, want_mask=True)
    bad, near, flipped = compare_masks(_np(gmask.active), mask, sc, 0.12)
    assert bad == 0
    ok_rows = ~rows_with_near(sc, 0.12)
    assert np.array_equal(_np(plan.counts)[ok_rows], counts[ok_rows])
    tri = np.broadcast_to(np.tril(np.ones(sc.shape[2:], bool)), sc.shape)
    rs = np.abs(_np(smap.score) - sc) / np.maximum(sc, 1e-30)
    assert rs[tri & (sc > 1e-6)].max() <= 1e-3


def test_discover_select_300k_tokens(fp):
    """Beyond the shared-memory row limit (M = 2344 key blocks): plan invariants of the reference
    (selection.hpp:176-192): ascending indices, fill N, 1 <= C <= i+1, sinks + window kept."""
    L, Hq, Hkv = 300_000, 2, 1
    q, k, _ = fp.workload.composite(3, 1, Hq, Hkv, L, device="cuda")
    plan = fp.discover_select(q, k, fp.PipelineConfig(alpha=0.12))[0]
    M = (L + 127) // 128
    idx = plan.indices[0].permute(2, 0, 1)  # h, i, slot
    cnt = plan.counts[0].permute(1, 0)       # h, i
    ar = torch.arange(M, device="cuda")
    assert bool((cnt >= 1).all()) and bool((cnt <= ar + 1).all())
    slots = torch.arange(M, device="cuda")[None, None, :]
    live = slots < cnt[:, :, None]
    assert bool((idx[~live] == M).all())
    nxt = torch.where(live[:, :, 1:], idx[:, :, 1:], torch.full_like(idx[:, :, 1:], M + 1))
    assert bool((nxt > idx[:, :, :-1]).all())
    for i in (0, 5, M // 2, M - 1):  # the diagonal block (window) and block 0 (sink) are kept
        row = idx[:, i, :]
        assert bool((row == i).any(dim=1).all()) and bool((row[:, 0] == 0).all())


@pytest.mark.parametrize("cfgv", [
    dict(sink_tokens=0, window_tokens=1, alpha=0.12),        # no structural retention
    dict(sink_tokens=1000, window_tokens=129, alpha=0.2),    # ceil-derived 8 sink / 2 window blocks
    dict(sink_tokens=256, window_tokens=2000, alpha=0.05),   # wide window
    dict(sink_tokens=256, window_tokens=512, alpha=0.12, scale=0.05),  # explicit tau
    dict(sink_tokens=256, window_tokens=512, alpha=0.12, epsilon=1e-3),
])
@pytest.mark.parametrize("shape", [(1, 3, 1, 1537), (2, 6, 3, 777), (1, 2, 2, 100)])
def test_config_variants_pipeline(fp, port, cfgv, shape):
    """PipelineConfig variants (core.hpp:87-112) through the fused path and attention: masks
    bit-exact outside the epsilon band, attention within the bf16 bars on the same plan; includes
    non-power-of-two GQA (6 Q / 3 KV heads), ragged L and a single partial block (L = 100)."""
    Z, Hq, Hkv, L = shape
    q, k, v = (bf16_round(x) for x in composite_np(41 + L, Z, Hq, Hkv, L))
    cfg = fp.PipelineConfig(**cfgv)
    tau = float(cfg.resolved_scale(128))
    eps = cfgv.get("epsilon", 1e-10)
    kk = np.repeat(k, Hq // Hkv, axis=1)  # the oracle has no GQA: per-Q-head K
    vv = np.repeat(v, Hq // Hkv, axis=1)
    _, _, sc = port.discover(q, kk, 128, tau, eps)
    mask, _ = port.max_threshold_mask(sc, 128, cfg.alpha, cfg.sink_tokens, cfg.window_tokens)
    plan, _, gmask = fp.discover_select(_cuda(q), _cuda(k), cfg, want_mask=True)
    bad, near, flipped = compare_masks(_np(gmask.active), mask, sc, cfg.alpha)
    assert bad == 0, (bad, near, flipped)
    gi, gc = _np(plan.indices), _np(plan.counts)
    ro, rl, _ = port.block_sparse_attention(q, kk, vv, gi, gc, 128, tau)
    res = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v), plan,
                                    fp.make_block_grid(L, 128), tau, out_dtype=torch.float32)
    _attn_check(_np(res.out), _np(res.lse), ro, rl)


# --------------------------------------------------------------------------- attention (K4/K5)
def _attn_check(go, gl, ro, rl):
    mx, mean = err(go, ro)
    lmx, lmean = err(gl, rl)
    print(f"out max {mx:.3e} mean {mean:.3e} | lse max {lmx:.3e} mean {lmean:.3e}")
    assert mx <= OUT_MAX_ABS and mean <= OUT_MEAN_ABS
    assert lmx <= OUT_MAX_ABS and lmean <= OUT_MEAN_ABS


@pytest.mark.parametrize("shape", [(1, 2, 2, 1024), (1, 4, 2, 1000), (2, 2, 1, 640),
                                   (1, 1, 1, 130)])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_sparse_attention_same_plan(fp, port, shape, out_dtype):
    Z, Hq, Hkv, L = shape
    q, k, v = (bf16_round(x) for x in composite_np(7 + L, Z, Hq, Hkv, L))
    tau = float(port.scale(128))
    _, _, sc = port.discover(q, k, 128, tau)
    mask, _ = port.max_threshold_mask(sc, 128, 0.12, 256, 512)
    idx, counts = port.compress_indices(mask)
    ro, rl, rvis = port.block_sparse_attention(q, k, v, idx, counts, 128, tau)
    st = fp.AttentionStats()
    res = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v),
                                    fp.SparseBlockPlan(_cuda(idx, torch.int32),
                                                       _cuda(counts, torch.int32)),
                                    fp.make_block_grid(L, 128), tau, st, out_dtype=out_dtype)
    assert st.block_visits == rvis
    _attn_check(_np(res.out), _np(res.lse), ro, rl)


@pytest.mark.parametrize("L", [128, 700, 1024, 2048])
def test_dense_attention(fp, port, L):
    q, k, v = (bf16_round(x) for x in composite_np(L, 1, 2, 1, L))
    tau = float(port.scale(128))
    ro, rl = port.dense_attention(q, k, v, tau)
    res = fp.dense_attention(_cuda(q), _cuda(k), _cuda(v), tau, out_dtype=torch.float32)
    _attn_check(_np(res.out), _np(res.lse), ro, rl)


def test_full_plan_equals_dense(fp, port):
    L = 1500
    q, k, v = (bf16_round(x) for x in composite_np(2, 1, 2, 2, L))
    tau = float(port.scale(128))
    grid = fp.make_block_grid(L, 128)
    plan = fp.full_causal_plan(1, 2, grid)
    idx, counts = port.full_causal_plan(1, 2, grid.num_query_blocks)
    assert np.array_equal(_np(plan.indices), idx) and np.array_equal(_np(plan.counts), counts)
    a = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v), plan, grid, tau,
                                  out_dtype=torch.float32)
    b = fp.dense_attention(_cuda(q), _cuda(k), _cuda(v), tau, out_dtype=torch.float32)
    assert err(_np(a.out), _np(b.out))[0] <= 1e-4 and err(_np(a.lse), _np(b.lse))[0] <= 1e-4


def test_attention_edge_semantics(fp, port):
    """count=0 -> NaN / -inf; listed j > i attended in full; PlanError on bad index."""
    L = 512
    q, k, v = (bf16_round(x) for x in composite_np(9, 1, 1, 1, L))
    tau = float(port.scale(128))
    M = 4
    idx = np.full((1, M, M, 1), M, np.int32)
    counts = np.zeros((1, M, 1), np.int32)
    idx[0, 0, :2, 0] = [0, 3]   # row 0 lists a future block (attended in full)
    counts[0, 0, 0] = 2
    idx[0, 2, :1, 0] = [1]      # row 2 without its diagonal
    counts[0, 2, 0] = 1
    # rows 1 and 3 empty -> NaN / -inf
    ro, rl, _ = port.block_sparse_attention(q, k, v, idx, counts, 128, tau)
    res = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v),
                                    fp.SparseBlockPlan(_cuda(idx, torch.int32),
                                                       _cuda(counts, torch.int32)),
                                    fp.make_block_grid(L, 128), tau, out_dtype=torch.float32)
    go, gl = _np(res.out), _np(res.lse)
    assert np.array_equal(np.isnan(go), np.isnan(ro))
    assert np.array_equal(np.isneginf(gl), np.isneginf(rl))
    fin = ~np.isnan(ro)
    assert np.abs(go[fin] - ro[fin]).max() <= OUT_MAX_ABS
    fin = np.isfinite(rl)
    assert np.abs(gl[fin] - rl[fin]).max() <= OUT_MAX_ABS
    bad = idx.copy()
    bad[0, 0, 1, 0] = M  # fill value inside the counted prefix -> PlanError
    with pytest.raises(fp.PlanError):
        fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v),
                                  fp.SparseBlockPlan(_cuda(bad, torch.int32),
                                                     _cuda(counts, torch.int32)),
                                  fp.make_block_grid(L, 128), tau)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_many_empty_rows_interleaved_with_long_rows(fp, port, out_dtype):
    """Plans where most rows are empty (C = 0 -> NaN / -inf) between long rows: empty rows are
    written by the scheduler warp and never become work items, so a fast-finishing empty item
    cannot release plan-row buffers the producer is still reading (repeated launches)."""
    Z, H, L = 1, 3, 4096
    q, k, v = (bf16_round(x) for x in composite_np(13, Z, H, H, L))
    tau = float(port.scale(128))
    M = L // 128
    rng = np.random.default_rng(0)
    idx = np.full((Z, M, M, H), M, np.int32)
    counts = np.zeros((Z, M, H), np.int32)
    for h in range(H):
        for i in range(M):
            if rng.random() < 0.3:  # ~30% of rows have work, the rest are empty
                js = np.sort(rng.choice(i + 1, size=min(i + 1, int(rng.integers(1, 20))),
                                        replace=False))
                idx[0, i, :len(js), h] = js
                counts[0, i, h] = len(js)
    ro, rl, _ = port.block_sparse_attention(q, k, v, idx, counts, 128, tau)
    plan = fp.SparseBlockPlan(_cuda(idx, torch.int32), _cuda(counts, torch.int32))
    for _ in range(5):
        res = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v), plan,
                                        fp.make_block_grid(L, 128), tau, out_dtype=out_dtype)
        go, gl = _np(res.out), _np(res.lse)
        assert np.array_equal(np.isnan(go), np.isnan(ro))
        assert np.array_equal(np.isneginf(gl), np.isneginf(rl))
        fin = ~np.isnan(ro)
        assert np.abs(go[fin] - ro[fin]).max() <= OUT_MAX_ABS


def test_fp32_pipeline_c1_small(fp, port):
    """fp32 inputs (config C1 style, reduced L): discovery split-precision + attention."""
    L = 2048
    q, k, v = composite_np(1, 1, 1, 1, L)
    tau = float(port.scale(128))
    _, _, sc = port.discover(q, k, 128, tau)
    mask, _ = port.max_threshold_mask(sc, 128, 0.12, 256, 512)
    idx, counts = port.compress_indices(mask)
    cfg = fp.PipelineConfig()
    plan, _, gmask = fp.discover_select(_cuda(q, torch.float32), _cuda(k, torch.float32), cfg,
                                        want_mask=True)
    bad, near, _ = compare_masks(_np(gmask.active), mask, sc, 0.12)
    assert bad == 0
    ro, rl, _ = port.block_sparse_attention(q, k, v, idx, counts, 128, tau)
    res = fp.block_sparse_attention(_cuda(q, torch.float32), _cuda(k, torch.float32),
                                    _cuda(v, torch.float32),
                                    fp.SparseBlockPlan(_cuda(idx, torch.int32),
                                                       _cuda(counts, torch.int32)),
                                    fp.make_block_grid(L, 128), tau)
    _attn_check(_np(res.out), _np(res.lse), ro, rl)


def test_prefill_host_e2e(fp, port):
    L = 2048
    q, k, v = (bf16_round(x) for x in composite_np(21, 1, 4, 2, L))
    tau = float(port.scale(128))
    cfg = fp.PipelineConfig()
    qh, kh, vh = (torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in (q, k, v))
    out = torch.empty(qh.shape, dtype=torch.float32).pin_memory()
    lse = torch.empty(qh.shape[:3], dtype=torch.float32).pin_memory()
    M = (L + 127) // 128
    idx = torch.empty((1, M, M, 4), dtype=torch.int32)
    counts = torch.empty((1, M, 4), dtype=torch.int32)
    vis = fp.prefill_host(qh, kh, vh, cfg, out, lse, idx, counts)
    assert vis == int(counts.sum())
    ro, rl, rvis = port.block_sparse_attention(q, k, v, idx.numpy(), counts.numpy(), 128, tau)
    assert rvis == vis
    _attn_check(out.numpy(), lse.numpy(), ro, rl)


@pytest.mark.parametrize("chunks", ["1", "3", "16"])
def test_prefill_host_rows_equal_device(fp, monkeypatch, chunks):
    """The row-chunked host pipeline (H2D of each chunk's token rows of every head, pooling,
    discovery and attention of those rows, D2H) reproduces the device-resident calls bit for bit:
    plan, output and LSE, including a ragged last block and Z = 2."""
    monkeypatch.setenv("FPB_E2E_CHUNKS", chunks)
    Z, Hq, Hkv, L = 2, 4, 2, 3000
    q, k, v = fp.workload.composite(31, Z, Hq, Hkv, L)
    cfg = fp.PipelineConfig(alpha=0.1)
    grid = fp.make_block_grid(L, 128)
    qd, kd, vd = (x.cuda() for x in (q, k, v))
    plan = fp.discover_select(qd, kd, cfg)[0]
    res = fp.block_sparse_attention(qd, kd, vd, plan, grid, cfg.resolved_scale(128),
                                    out_dtype=torch.bfloat16)
    qh, kh, vh = (x.pin_memory() for x in (q, k, v))
    out = torch.empty(qh.shape, dtype=torch.bfloat16).pin_memory()
    lse = torch.empty(qh.shape[:3], dtype=torch.float32).pin_memory()
    M = grid.num_query_blocks
    idx = torch.empty((Z, M, M, Hq), dtype=torch.int32)
    counts = torch.empty((Z, M, Hq), dtype=torch.int32)
    vis = fp.prefill_host(qh, kh, vh, cfg, out, lse, idx, counts)
    assert torch.equal(counts, plan.counts.cpu()) and torch.equal(idx, plan.indices.cpu())
    assert vis == int(counts.to(torch.int64).sum())
    assert torch.equal(out, res.out.cpu()) and torch.equal(lse, res.lse.cpu())


# --------------------------------------------------------------------------- committed goldens
def _golden_cases():
    import glob
    import os
    return sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "gpu_*.npz")))


@pytest.mark.parametrize("path", _golden_cases())
def test_golden_reference_vectors(fp, port, path):
    """CUDA path vs outputs produced by the unmodified reference (tests/golden/gen_golden.py)."""
    g = np.load(path)
    kind, strength, a, b, noise, seed, Z, H, L, d, B, bf = g["params"]
    q, k, v, _ = port.generate_planted(int(kind), float(strength), int(a), int(b), float(noise),
                                       int(seed), int(Z), int(H), int(L), int(d), int(B))
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    L = int(L)
    grid = fp.make_block_grid(L, 128)
    tau = float(port.scale(128))
    assert np.array_equal(_np(fp.pool_keys(_cuda(k), grid).data), g["pooled"])
    for al in (0.0, 0.12, 0.5):
        tag = f"a{int(al * 100):03d}"
        plan, smap, gm = fp.discover_select(_cuda(q), _cuda(k), fp.PipelineConfig(alpha=al),
                                            want_score=True, want_mask=True)
        bad, near, _ = compare_masks(_np(gm.active), g[f"mask_{tag}"], g["score"], al)
        assert bad == 0
        ok = ~rows_with_near(g["score"], al)
        assert np.array_equal(_np(plan.counts)[ok], g[f"counts_{tag}"][ok])
        # standalone threshold/compaction on the reference's own score map: bit-exact
        st = fp.SelectionStats()
        m2 = fp.max_threshold_mask(_cuda(g["score"], torch.float32), fp.PipelineConfig(alpha=al), st)
        assert np.array_equal(_np(m2.active), g[f"mask_{tag}"])
        assert st.score_comparisons == int(g[f"cmp_{tag}"][0])
        p2 = fp.compress_indices(m2)
        assert np.array_equal(_np(p2.indices), g[f"idx_{tag}"])
        assert np.array_equal(_np(p2.counts), g[f"counts_{tag}"])
    st = fp.AttentionStats()
    res = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v),
                                    fp.SparseBlockPlan(_cuda(g["idx_a012"], torch.int32),
                                                       _cuda(g["counts_a012"], torch.int32)),
                                    grid, tau, st, out_dtype=torch.float32)
    assert st.block_visits == int(g["visits"][0])
    _attn_check(_np(res.out), _np(res.lse), g["out_sparse"], g["lse_sparse"])
    if "out_dense" in g.files:
        res = fp.dense_attention(_cuda(q), _cuda(k), _cuda(v), tau, out_dtype=torch.float32)
        _attn_check(_np(res.out), _np(res.lse), g["out_dense"], g["lse_dense"])


# --------------------------------------------------------------------------- full-size properties
def test_qwen3_32k_plan_invariants_and_full_plan_identity(fp):
    """BASELINE config 2 at full size: plan invariants (selection.hpp:176-192 + :53-56) and the
    size-independent identity sparse(full causal plan) == dense (acceptance.cpp crit. 1)."""
    from paper_2603_06199_b200 import workload
    L = 32768
    q, k, v = (x.cuda() for x in workload.qwen3_30b_a3b(L, seed=3))
    cfg = fp.PipelineConfig()
    plan, _, mask = fp.discover_select(q, k, cfg, want_mask=True)
    M = L // 128
    idx, counts = plan.indices.long(), plan.counts.long()
    slot = torch.arange(M, device="cuda").view(1, 1, M, 1)
    within = slot < counts.view(1, M, 1, 32)
    # strictly increasing active prefix, fill value N after it, counts in [min retained, i+1]
    assert torch.all((idx[..., :-1, :] < idx[..., 1:, :]) | ~within[..., 1:, :])
    assert torch.all(torch.where(within, True, idx == M))
    i = torch.arange(M, device="cuda").view(1, M, 1)
    assert torch.all(counts <= i + 1) and torch.all(counts >= torch.clamp(i + 1, max=6))
    # mask <-> plan round trip, and retention of sink / window / diagonal blocks
    assert torch.equal(mask.active.sum(dim=2).long(), counts)
    diag = mask.active[0, torch.arange(M), torch.arange(M), :]
    assert torch.all(diag == 1)
    assert torch.all(mask.active[0, 2:, :2, :] == 1)
    grid = fp.make_block_grid(L, 128)
    tau = cfg.resolved_scale(128)
    full = fp.full_causal_plan(1, 32, grid)
    a = fp.block_sparse_attention(q, k, v, full, grid, tau, out_dtype=torch.float32)
    b = fp.dense_attention(q, k, v, tau, out_dtype=torch.float32)
    assert torch.equal(a.out, b.out) and torch.equal(a.lse, b.lse)
    st = fp.AttentionStats()
    fp.block_sparse_attention(q, k, v, plan, grid, tau, st)
    assert st.block_visits == int(counts.sum())


def test_misaligned_views_rejected(fp):
    """The tcgen05 path moves Q / K / V / O with TMA and bulk copies: a tensor whose base address
    is not 16-byte aligned (a 2-byte-offset view) is a ValidationError, not a device fault."""
    L = 1024
    q, k, v = (x.cuda() for x in fp.workload.composite(3, 1, 2, 1, L))
    cfg = fp.PipelineConfig()

    def shifted(t):  # same shape, base address + 2 bytes
        flat = torch.empty(t.numel() + 8, dtype=t.dtype, device=t.device)
        view = flat[1:1 + t.numel()].view(t.shape)
        view.copy_(t)
        return view

    with pytest.raises(fp.ValidationError):
        fp.discover_select(shifted(q), k, cfg)
    with pytest.raises(fp.ValidationError):
        fp.discover_select(q, shifted(k), cfg)
    plan = fp.discover_select(q, k, cfg)[0]
    grid = fp.make_block_grid(L, 128)
    with pytest.raises(fp.ValidationError):
        fp.block_sparse_attention(q, k, shifted(v), plan, grid, cfg.resolved_scale(128))
    with pytest.raises(fp.ValidationError):
        fp.pool_keys(shifted(k), grid)
    torch.cuda.synchronize()  # the context is still healthy
    res = fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128))
    assert torch.isfinite(res.lse).all()


def test_prefill_host_concurrent_threads(fp):
    """fpb_host_prefill keeps a per-thread device arena and streams: two host threads calling it at
    once (ctypes releases the GIL) get the same results as sequential calls."""
    import threading
    L = 3000
    ins = [fp.workload.composite(61 + i, 1, 4, 2, L) for i in range(2)]
    cfg = fp.PipelineConfig()

    def run(i, res):
        q, k, v = (x.pin_memory() for x in ins[i])
        out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
        lse = torch.empty(q.shape[:3], dtype=torch.float32).pin_memory()
        for _ in range(3):
            fp.prefill_host(q, k, v, cfg, out, lse)
        res[i] = (out.clone(), lse.clone())

    seq = {}
    for i in range(2):
        run(i, seq)
    par = {}
    ts = [threading.Thread(target=run, args=(i, par)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        assert torch.equal(par[i][0], seq[i][0]) and torch.equal(par[i][1], seq[i][1])
