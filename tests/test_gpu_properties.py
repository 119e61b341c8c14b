"""GPU: the reference's attention property tests (test_attention.cpp:158-236) and acceptance
criterion 1 (acceptance.cpp:59-109), restated on the tcgen05 path (d = B = 128, bf16 inputs,
fp32 output so the properties are not hidden by output rounding).

  * block order: a plan row's list in any order gives the same result (LSE within 1e-4, output
    within the bf16 bars: P is rounded to bf16 against an order-dependent running max);
  * monotone LSE: adding blocks to a row never lowers its log-sum-exp;
  * convex hull: every output channel lies within the [min, max] of V over the attended keys;
  * 20 random shapes (L, Hq, Hkv incl. GQA and ragged L): full causal plan == dense within 1e-4;
  * discovery KATs (test_discovery.cpp:70-134): identical query rows, energy bound, sentinels;
  * selection: alpha-monotone plans, alpha = 0 keeps every causal block (test_selection.cpp).
"""
import numpy as np
import pytest
import torch

from tests._util import OUT_MAX_ABS, OUT_MEAN_ABS, bf16_round, composite_np, err

pytestmark = pytest.mark.gpu


def _cuda(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _np(t):
    return t.detach().cpu().numpy() if t.dtype == torch.int32 else t.float().cpu().numpy()


def _layer(seed, Hq, Hkv, L):
    q, k, v = (bf16_round(x) for x in composite_np(seed, 1, Hq, Hkv, L))
    return q, k, v


def _attend(fp, q, k, v, idx, counts, L, tau):
    plan = fp.SparseBlockPlan(_cuda(idx, torch.int32), _cuda(counts, torch.int32))
    res = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v), plan, fp.make_block_grid(L, 128),
                                    tau, out_dtype=torch.float32)
    return _np(res.out), _np(res.lse)


def _random_plan(rng, M, H, p=0.4):
    """Causal rows with the diagonal always listed, ascending (the reference's plan form)."""
    idx = np.full((1, M, M, H), M, np.int32)
    counts = np.zeros((1, M, H), np.int32)
    for i in range(M):
        for h in range(H):
            js = [j for j in range(i) if rng.random() < p] + [i]
            idx[0, i, :len(js), h] = js
            counts[0, i, h] = len(js)
    return idx, counts


def test_block_order_invariance(fp, port):
    """test_attention.cpp:167-183: the online softmax makes the visit order irrelevant (<= 1e-4)."""
    L, Hq, Hkv = 2000, 4, 2
    q, k, v = _layer(41, Hq, Hkv, L)
    tau = float(port.scale(128))
    M = -(-L // 128)
    rng = np.random.default_rng(3)
    idx, counts = _random_plan(rng, M, Hq)
    o1, l1 = _attend(fp, q, k, v, idx, counts, L, tau)
    shuf = idx.copy()
    for i in range(M):
        for h in range(Hq):
            c = counts[0, i, h]
            shuf[0, i, :c, h] = rng.permutation(idx[0, i, :c, h])  # descending, random, ...
    o2, l2 = _attend(fp, q, k, v, shuf, counts, L, tau)
    eo, el = err(o1, o2), err(l1, l2)
    print(f"order: out max/mean {eo}, lse max/mean {el}")
    # P enters the PV MMA as bf16 relative to the running row max, which depends on the order:
    # the order-invariance holds to the bf16 bars (the reference's fp32 P gives 1e-4); the LSE
    # (fp32 row sums of the unrounded P) stays at the reference's 1e-4
    assert eo[0] <= OUT_MAX_ABS and eo[1] <= OUT_MEAN_ABS and el[0] <= 1e-4


def test_lse_monotone_in_visited_blocks(fp, port):
    """test_attention.cpp:185-210: a superset plan row has an LSE at least as large."""
    L, Hq, Hkv = 1800, 2, 1
    q, k, v = _layer(43, Hq, Hkv, L)
    tau = float(port.scale(128))
    M = -(-L // 128)
    rng = np.random.default_rng(5)
    idx_a, cnt_a = _random_plan(rng, M, Hq, p=0.3)
    idx_b, cnt_b = idx_a.copy(), cnt_a.copy()
    for i in range(M):  # add every remaining causal block, keep ascending order
        for h in range(Hq):
            js = list(range(i + 1))
            idx_b[0, i, :len(js), h] = js
            cnt_b[0, i, h] = len(js)
    _, la = _attend(fp, q, k, v, idx_a, cnt_a, L, tau)
    _, lb = _attend(fp, q, k, v, idx_b, cnt_b, L, tau)
    assert np.all(lb >= la - 1e-4), float((la - lb).max())


def test_output_in_convex_hull_of_values(fp, port):
    """test_attention.cpp:212-236: softmax weights are a convex combination, so every output
    channel lies in [min, max] of that channel of V over the keys the row attends."""
    L, Hq, Hkv = 1100, 2, 2
    q, k, v = _layer(47, Hq, Hkv, L)
    tau = float(port.scale(128))
    M = -(-L // 128)
    rng = np.random.default_rng(9)
    idx, counts = _random_plan(rng, M, Hq, p=0.5)
    out, _ = _attend(fp, q, k, v, idx, counts, L, tau)
    for h in range(Hq):
        for i in range(M):
            rows = range(i * 128, min(L, (i + 1) * 128))
            blocks = idx[0, i, :counts[0, i, h], h]
            for r in rows:
                keys = np.concatenate([np.arange(j * 128, min(L, (j + 1) * 128, r + 1 if j == i
                                                              else L)) for j in blocks])
                vk = v[0, h // (Hq // Hkv), keys]
                o = out[0, h, r]
                assert np.all(o >= vk.min(axis=0) - 1e-5) and np.all(o <= vk.max(axis=0) + 1e-5)


_SHAPES = [(int(L), int(H), int(H // g)) for L, H, g in zip(
    np.random.default_rng(2024).integers(100, 3000, 20),
    np.random.default_rng(7).choice([1, 2, 4, 6, 8], 20),
    np.random.default_rng(8).choice([1, 2], 20)) if H % g == 0] + [(128, 1, 1), (129, 2, 1)]


@pytest.mark.parametrize("L,Hq,Hkv", _SHAPES[:20])
def test_acceptance_full_plan_equals_dense(fp, port, L, Hq, Hkv):
    """acceptance.cpp:59-109 (criterion 1): on random shapes the sparse kernel with the full causal
    plan equals the dense kernel within 1e-4, and the plan equals the oracle's full plan."""
    q, k, v = _layer(L + Hq, Hq, Hkv, L)
    tau = float(port.scale(128))
    grid = fp.make_block_grid(L, 128)
    plan = fp.full_causal_plan(1, Hq, grid)
    idx, counts = port.full_causal_plan(1, Hq, grid.num_query_blocks)
    assert np.array_equal(_np(plan.indices), idx) and np.array_equal(_np(plan.counts), counts)
    a = fp.block_sparse_attention(_cuda(q), _cuda(k), _cuda(v), plan, grid, tau,
                                  out_dtype=torch.float32)
    b = fp.dense_attention(_cuda(q), _cuda(k), _cuda(v), tau, out_dtype=torch.float32)
    assert err(_np(a.out), _np(b.out))[0] <= 1e-4 and err(_np(a.lse), _np(b.lse))[0] <= 1e-4


def test_discovery_identical_rows_kat(fp, port):
    """test_discovery.cpp:70-89: when every query row of a block is the same vector q, each
    causal pair's local max is the scaled logit q . k̄_J and its energy is the row count (all
    exp2 terms are 1); the ragged last block counts its real rows only."""
    L, d = 300, 128
    rng = np.random.default_rng(1)
    qrow = bf16_round(rng.normal(size=(d,)).astype(np.float32))
    q = np.broadcast_to(qrow, (1, 1, L, d)).copy()
    k = bf16_round(rng.normal(size=(1, 1, L, d)).astype(np.float32))
    tau = float(port.scale(d))
    m = fp.discover(_cuda(q), _cuda(k), fp.make_block_grid(L, 128), tau)
    en, lm = _np(m.energy)[0, 0], _np(m.local_max)[0, 0]
    pooled = port.pool_keys(k, 128)[0, 0]
    M = -(-L // 128)
    for I in range(M):
        rows = min(128, L - I * 128)
        for J in range(I + 1):
            want = float(np.dot(qrow.astype(np.float64), pooled[J].astype(np.float64))) * \
                tau * 1.4426950408889634
            assert abs(lm[I, J] - want) <= 1e-4 * max(1.0, abs(want))
            assert abs(en[I, J] - rows) <= 1e-3 * rows


def test_discovery_energy_bound_and_sentinels(fp, port):
    """test_discovery.cpp:91-134: 0 < S_IJ <= rows of block I for causal pairs; J > I holds the
    sentinels (energy 0, local max FLT_LOWEST, score 0); each score row sums to ~1."""
    L = 1500
    q, k, _ = _layer(51, 2, 1, L)
    tau = float(port.scale(128))
    m = fp.discover(_cuda(q), _cuda(k), fp.make_block_grid(L, 128), tau)
    en, lm, sc = _np(m.energy), _np(m.local_max), _np(m.score)
    M = en.shape[2]
    tri = np.tril(np.ones((M, M), bool))
    rows = np.array([min(128, L - I * 128) for I in range(M)], np.float32)[:, None]
    for h in range(2):
        e = en[0, h]
        assert np.all(e[tri] > 0) and np.all((e <= rows * (1 + 1e-6))[tri])
        assert np.all(e[~tri] == 0) and np.all(sc[0, h][~tri] == 0)
        assert np.all(lm[0, h][~tri] == np.finfo(np.float32).min)
        assert np.allclose(sc[0, h].sum(axis=1), 1.0, atol=1e-5)


def test_selection_alpha_monotone(fp):
    """test_selection.cpp:58-120: a larger alpha never activates a block a smaller one drops
    (plans nest), and alpha = 0 keeps every causal block."""
    L = 4096
    q, k, _ = _layer(53, 4, 2, L)
    M = L // 128
    prev = None
    for alpha in (0.0, 0.05, 0.12, 0.3, 1.0):
        _, _, gm = fp.discover_select(_cuda(q), _cuda(k), fp.PipelineConfig(alpha=alpha),
                                      want_mask=True)
        mask = _np(gm.active).astype(bool)
        if alpha == 0.0:
            tri = np.tril(np.ones((M, M), bool))[None, :, :, None]
            assert np.array_equal(mask, np.broadcast_to(tri, mask.shape))
        if prev is not None:
            assert not np.any(mask & ~prev)
        prev = mask
