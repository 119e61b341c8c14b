"""GPU: the SIMT path for shapes outside the tensor-core tile (d != 128 or B != 128), against the
oracle at the reference's own test shapes.  Logits/maxima/pooled keys follow the reference's
arithmetic order exactly, so local_max and pooled keys are bit-identical; only exp2f/log2f may
differ by a few ulp."""
import numpy as np
import pytest
import torch

from tests._util import compare_masks, err, rows_with_near

pytestmark = pytest.mark.gpu

SHAPES = [(256, 32, 16, 2), (130, 64, 8, 1), (47, 16, 4, 3), (1000, 128, 32, 2), (777, 64, 64, 2)]


def _t(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _n(t):
    return t.detach().cpu().numpy() if t.dtype in (torch.uint8, torch.int32) else t.float().cpu().numpy()


@pytest.mark.parametrize("L,B,d,H", SHAPES)
def test_generic_full_plan_equals_dense(fp, port, L, B, d, H):
    """test_attention.cpp:67-83 / acceptance crit. 1: sparse(full plan) == dense within 1e-4."""
    rng = np.random.default_rng(100 + L)
    q, k, v = (rng.normal(size=(1, H, L, d)).astype(np.float32) for _ in range(3))
    tau = float(port.scale(d))
    grid = fp.make_block_grid(L, B)
    plan = fp.full_causal_plan(1, H, grid)
    st = fp.AttentionStats()
    a = fp.block_sparse_attention(_t(q), _t(k), _t(v), plan, grid, tau, st)
    b = fp.dense_attention(_t(q), _t(k), _t(v), tau)
    assert err(_n(a.out), _n(b.out))[0] <= 1e-4 and err(_n(a.lse), _n(b.lse))[0] <= 1e-4
    assert st.block_visits == grid.num_query_blocks * (grid.num_query_blocks + 1) // 2 * H
    ro, rl = port.dense_attention(q, k, v, tau)
    assert err(_n(b.out), ro)[0] <= 1e-4 and err(_n(b.lse), rl)[0] <= 1e-4


@pytest.mark.parametrize("L,B,d,H", SHAPES)
def test_generic_pipeline_vs_oracle(fp, port, L, B, d, H):
    q, k, v, _ = port.generate_planted(1, 2.5, max(1, L // 3), 0, 0.5, 7, 1, H, L, d, B)
    tau = float(port.scale(d))
    grid = fp.make_block_grid(L, B)
    assert np.array_equal(_n(fp.pool_keys(_t(k), grid).data), port.pool_keys(k, B))
    en, lm, sc = port.discover(q, k, B, tau)
    m = fp.discover(_t(q), _t(k), grid, tau)
    assert np.array_equal(_n(m.local_max), lm)  # 4-lane dot order replicated: bit-exact
    assert np.allclose(_n(m.energy), en, rtol=1e-5, atol=0)
    assert np.allclose(_n(m.score), sc, rtol=1e-5, atol=1e-7)
    cfg = fp.PipelineConfig(block_size=B, alpha=0.12, sink_tokens=B, window_tokens=B)
    plan, _, gm = fp.discover_select(_t(q), _t(k), cfg, want_mask=True)
    mask, _ = port.max_threshold_mask(sc, B, 0.12, B, B)
    bad, near, _ = compare_masks(_n(gm.active), mask, sc, 0.12)
    assert bad == 0
    idx, counts = port.compress_indices(mask)
    ok = ~rows_with_near(sc, 0.12)
    assert np.array_equal(_n(plan.counts)[ok], counts[ok])
    ro, rl, rvis = port.block_sparse_attention(q, k, v, idx, counts, B, tau)
    st = fp.AttentionStats()
    res = fp.block_sparse_attention(_t(q), _t(k), _t(v),
                                    fp.SparseBlockPlan(_t(idx, torch.int32), _t(counts, torch.int32)),
                                    grid, tau, st)
    assert st.block_visits == rvis
    assert err(_n(res.out), ro)[0] <= 1e-5 and err(_n(res.lse), rl)[0] <= 1e-5
