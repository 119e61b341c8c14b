"""GPU: the reference's comparison baselines against the oracle.
top-k / top-p are bit-exact given the same score map (ties included); pool-both / exact discovery
reproduce local_max bit-for-bit (same 4-lane dot order) and energy / score within float ulps."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _t(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _n(t):
    return t.detach().cpu().numpy() if t.dtype in (torch.uint8, torch.int32) else t.float().cpu().numpy()


@pytest.mark.parametrize("M,H", [(1, 1), (7, 2), (33, 3), (200, 2)])
def test_topk_topp_bitexact(fp, port, M, H):
    rng = np.random.default_rng(M)
    sc = rng.random((2, H, M, M)).astype(np.float32)
    sc[..., ::4] = sc[..., :1]                          # ties -> lower index first
    sc[0, 0, -1, :] = 0.0                               # all-zero row for top-p
    B = 64
    cfg = fp.PipelineConfig(block_size=B, sink_tokens=64, window_tokens=128)
    for k in (1, 3, 8):
        got = _n(fp.topk_select(_t(sc), k, cfg).active)
        assert np.array_equal(got, port.sort_select(sc, "topk", k, B, 64, 128)), k
    for p in (0.3, 0.9, 1.0):
        got = _n(fp.topp_select(_t(sc), p, cfg).active)
        assert np.array_equal(got, port.sort_select(sc, "topp", p, B, 64, 128)), p
    with pytest.raises(fp.ConfigError):
        fp.topk_select(_t(sc), 0, cfg)
    with pytest.raises(fp.ConfigError):
        fp.topp_select(_t(sc), 1.5, cfg)


@pytest.mark.parametrize("method", ["pool-both", "exact"])
@pytest.mark.parametrize("L,B,d,Hq,Hkv", [(512, 64, 32, 2, 2), (1000, 128, 128, 4, 2),
                                          (300, 32, 16, 3, 1)])
def test_discover_baselines(fp, port, method, L, B, d, Hq, Hkv):
    rng = np.random.default_rng(L + d)
    q = rng.normal(size=(1, Hq, L, d)).astype(np.float32)
    k = rng.normal(size=(1, Hkv, L, d)).astype(np.float32)
    tau = float(port.scale(d))
    en, lm, sc = port.discover_variant(method, q, k, B, tau)
    fn = fp.discover_pool_both if method == "pool-both" else fp.discover_exact
    m = fn(_t(q), _t(k), fp.make_block_grid(L, B), tau)
    assert np.array_equal(_n(m.local_max), lm)
    assert np.allclose(_n(m.energy), en, rtol=2e-6, atol=0)
    assert np.allclose(_n(m.score), sc, rtol=2e-5, atol=1e-8)
