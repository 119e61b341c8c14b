"""CPU: pin the oracle (C restatement) against golden vectors from the reference itself, and
against the reference's own known-answer tests (restated with the same inputs / expectations).

Golden fixtures come from tests/golden/gen_golden.py run against the UNMODIFIED reference headers
(oracle/_ref).  Equality is bit-exact: the restatement keeps the reference's arithmetic order.
"""
import glob
import os

import numpy as np
import pytest

from oracle import LOG2E, NEG_SENTINEL

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if os.path.basename(p) != "cli.npz")  # cli.npz: CLI fixtures, tests/test_cli.py


def _inputs(port, P):
    kind, strength, a, b, noise, seed, Z, H, L, d, B, bf = P
    q, k, v, gt = port.generate_planted(int(kind), float(strength), int(a), int(b), float(noise),
                                        int(seed), int(Z), int(H), int(L), int(d), int(B))
    if bf:
        from tests._util import bf16_round
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v, gt, int(L), int(d), int(B)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_matches_reference_golden(port, path):
    g = np.load(path)
    q, k, v, gt, L, d, B = _inputs(port, g["params"])
    assert np.array_equal(g["q_sum"], [q.astype(np.float64).sum(), k.astype(np.float64).sum(),
                                       v.astype(np.float64).sum()])
    assert np.array_equal(gt, g["gt"])
    assert np.array_equal(port.pool_keys(k, B), g["pooled"])
    tau = float(port.scale(d))
    en, lm, sc = port.discover(q, k, B, tau)
    assert np.array_equal(en, g["energy"])
    assert np.array_equal(lm, g["local_max"])
    assert np.array_equal(sc, g["score"])
    for al in (0.0, 0.12, 0.5):
        tag = f"a{int(al * 100):03d}"
        mask, cmp = port.max_threshold_mask(sc, B, al, 256, 512)
        assert np.array_equal(mask, g[f"mask_{tag}"]) and cmp == int(g[f"cmp_{tag}"][0])
        idx, counts = port.compress_indices(mask)
        assert np.array_equal(idx, g[f"idx_{tag}"]) and np.array_equal(counts, g[f"counts_{tag}"])
        if al == 0.12:
            o, lse, vis = port.block_sparse_attention(q, k, v, idx, counts, B, tau)
            assert np.array_equal(o, g["out_sparse"]) and np.array_equal(lse, g["lse_sparse"])
            assert vis == int(g["visits"][0])
    if "out_dense" in g:
        o, lse = port.dense_attention(q, k, v, tau)
        assert np.array_equal(o, g["out_dense"]) and np.array_equal(lse, g["lse_dense"])
    if "topk4" in g:  # comparison baselines
        assert np.array_equal(port.sort_select(sc, "topk", 4, B, 256, 512), g["topk4"])
        assert np.array_equal(port.sort_select(sc, "topp", 0.9, B, 256, 512), g["topp09"])
        for name in ("pool-both", "exact"):
            tag = name.replace("-", "_")
            e2, l2, s2 = port.discover_variant(name, q, k, B, tau)
            assert np.array_equal(e2, g[f"{tag}_energy"]) and np.array_equal(l2, g[f"{tag}_local_max"])
            assert np.array_equal(s2, g[f"{tag}_score"])


def test_oracle_matches_live_reference(port, ref):
    """Random shapes / GQA-free configs: port == reference bit for bit (when _ref is built)."""
    rng = np.random.default_rng(0)
    for trial in range(6):
        L = int(rng.integers(8, 600))
        d = int(rng.integers(4, 40))
        B = int(rng.integers(4, 130))
        H = int(rng.integers(1, 3))
        q = rng.normal(size=(1, H, L, d)).astype(np.float32)
        k = rng.normal(size=(1, H, L, d)).astype(np.float32)
        v = rng.normal(size=(1, H, L, d)).astype(np.float32)
        tau = float(port.scale(d))
        a = port.discover(q, k, B, tau)
        b = ref.discover(q, k, B, tau)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        m1, c1 = port.max_threshold_mask(a[2], B, 0.2, 3 * B // 2, B + 1)
        m2, c2 = ref.max_threshold_mask(b[2], B, 0.2, 3 * B // 2, B + 1)
        assert np.array_equal(m1, m2) and c1 == c2
        i1, n1 = port.compress_indices(m1)
        o1 = port.block_sparse_attention(q, k, v, i1, n1, B, tau)
        o2 = ref.block_sparse_attention(q, k, v, i1, n1, B, tau)
        assert np.array_equal(o1[0], o2[0]) and np.array_equal(o1[1], o2[1]) and o1[2] == o2[2]


# ----------------------------------------------------------------- restated reference KATs
def test_kat_pool_hand_arithmetic(port):
    """test_discovery.cpp:24-35 and :53-60."""
    k = np.array([[[[1, 3], [3, 1]]]], np.float32)
    assert np.array_equal(port.pool_keys(k, 2), [[[[2, 2]]]])
    k = np.arange(5, dtype=np.float32).reshape(1, 1, 5, 1)
    p = port.pool_keys(k, 4)
    assert p[0, 0, 0, 0] == 1.5 and p[0, 0, 1, 0] == 4.0


def test_kat_identical_rows(port):
    """test_discovery.cpp:70-89: identical rows -> m = scaled logit, S = B."""
    B = 8
    q = np.tile(np.array([1, -2, 0.5], np.float32), (1, 1, B, 1))
    k = np.tile(np.array([0.25, 1, -1], np.float32), (1, 1, B, 1))
    tau = 0.5
    en, lm, _ = port.discover(q, k, B, tau)
    expected = np.float32(np.float32(1 * 0.25 - 2 * 1.0 + 0.5 * -1) * np.float32(tau) * LOG2E)
    assert lm[0, 0, 0, 0] == pytest.approx(expected, rel=1e-6) and en[0, 0, 0, 0] == B


def test_kat_sentinels_and_energy_bound(port):
    """test_discovery.cpp:91-101 and :120-134."""
    rng = np.random.default_rng(3)
    q = rng.normal(size=(2, 2, 21, 4)).astype(np.float32)
    k = rng.normal(size=(2, 2, 21, 4)).astype(np.float32)
    en, lm, sc = port.discover(q, k, 8, 0.5)
    M = 3
    for i in range(M):
        for j in range(M):
            if j > i:
                assert np.all(en[..., i, j] == 0) and np.all(lm[..., i, j] == NEG_SENTINEL)
                assert np.all(sc[..., i, j] == 0)
            else:
                rows = 5 if i == 2 else 8
                assert np.all(en[..., i, j] > 0) and np.all(en[..., i, j] <= rows * (1 + 1e-5))
                assert np.all(en[..., i, j] >= 1 - 1e-5)


def test_kat_threshold_hand_enumeration(port):
    """test_selection.cpp:59-75 and :111-119 (sink 0, window 1 token, B = 1)."""
    row = np.array([0.5, 0.3, 0.05, 0.15], np.float32)
    score = np.zeros((1, 1, 4, 4), np.float32)
    for i in range(4):
        score[0, 0, i, : i + 1] = row[: i + 1]

    def act(alpha):
        mask, cmp = port.max_threshold_mask(score, 1, alpha, 0, 1)
        return mask, cmp

    m, cmp = act(0.5)
    assert set(np.nonzero(m[0, 3, :, 0])[0]) == {0, 1, 3}
    assert cmp == 2 * 10
    m, _ = act(0.0)
    assert all(m[0, i, :, 0].sum() == i + 1 for i in range(4))
    m, _ = act(1.0)
    assert set(np.nonzero(m[0, 3, :, 0])[0]) == {0, 3}


def test_kat_compress(port):
    """test_selection.cpp:123-139."""
    mask = np.zeros((1, 1, 4, 1), np.uint8)
    mask[0, 0, [0, 2], 0] = 1
    idx, counts = port.compress_indices(mask)
    assert counts[0, 0, 0] == 2 and list(idx[0, 0, :, 0]) == [0, 2, 4, 4]


def test_kat_attention_basics(port):
    """test_attention.cpp:26-65."""
    q = np.zeros((1, 1, 2, 2), np.float32)
    q[0, 0, 1, 0] = 1
    k = np.zeros((1, 1, 2, 2), np.float32)
    k[0, 0, 0, 1] = 1
    v = np.zeros((1, 1, 2, 2), np.float32)
    v[0, 0, 0, 0] = 1
    v[0, 0, 1, 1] = 1
    idx, counts = port.full_causal_plan(1, 1, 1)
    o, lse, _ = port.block_sparse_attention(q, k, v, idx, counts, 2, 1.0)
    assert np.allclose(o[0, 0, 1], [0.5, 0.5]) and lse[0, 0, 1] == pytest.approx(1.0)
    # plan corruption -> PlanError (test_attention.cpp:238-258)
    q, k, v = (np.ones((1, 1, 8, 4), np.float32) for _ in range(3))
    idx, counts = port.full_causal_plan(1, 1, 2)
    idx[0, 1, 0, 0] = 2
    with pytest.raises(ValueError):
        port.block_sparse_attention(q, k, v, idx, counts, 4, 0.5)


def test_kat_full_plan_equals_dense(port):
    """test_attention.cpp:67-83 shapes (L, B, d, H) with 1e-4 tolerance."""
    rng = np.random.default_rng(4)
    for L, B, d, H in [(256, 32, 16, 2), (130, 64, 8, 1), (47, 16, 4, 3)]:
        q, k, v = (rng.normal(size=(1, H, L, d)).astype(np.float32) for _ in range(3))
        tau = float(port.scale(d))
        M = (L + B - 1) // B
        idx, counts = port.full_causal_plan(1, H, M)
        o, lse, vis = port.block_sparse_attention(q, k, v, idx, counts, B, tau)
        od, ld = port.dense_attention(q, k, v, tau)
        assert np.abs(o - od).max() <= 1e-4 and np.abs(lse - ld).max() <= 1e-4
        assert vis == port.visit_count(counts)


def test_gqa_equals_per_head_calls(port):
    """The GQA generalisation equals per-Q-head reference calls with the KV head's slice."""
    rng = np.random.default_rng(8)
    L, d, B = 300, 16, 64
    q = rng.normal(size=(1, 4, L, d)).astype(np.float32)
    k = rng.normal(size=(1, 2, L, d)).astype(np.float32)
    v = rng.normal(size=(1, 2, L, d)).astype(np.float32)
    tau = float(port.scale(d))
    en, lm, sc = port.discover(q, k, B, tau)
    mask, _ = port.max_threshold_mask(sc, B, 0.1, 64, 64)
    idx, counts = port.compress_indices(mask)
    o, lse, _ = port.block_sparse_attention(q, k, v, idx, counts, B, tau)
    for h in range(4):
        kh = h // 2
        e1, l1, s1 = port.discover(q[:, h:h + 1], k[:, kh:kh + 1], B, tau)
        assert np.array_equal(s1[0, 0], sc[0, h])
        o1, ls1, _ = port.block_sparse_attention(q[:, h:h + 1], k[:, kh:kh + 1], v[:, kh:kh + 1],
                                                 idx[..., h:h + 1], counts[..., h:h + 1], B, tau)
        assert np.array_equal(o1[0, 0], o[0, h]) and np.array_equal(ls1[0, 0], lse[0, h])
