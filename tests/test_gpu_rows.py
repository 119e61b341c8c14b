"""GPU: the row-sharded partition (fpb_discover_select_rows / fpb_block_sparse_attention_rows).

Every (z, h, query block) is independent through discovery, selection and attention
(discovery.hpp:87-88, selection.hpp:71-72, attention.hpp:59-60), so a rank that owns query blocks
r, r + G, ... must produce exactly the plan rows and output rows of the unsharded call: the same
kernels run the same per-item arithmetic, so the bar is bit-equality.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_row_shards_equal_whole(fp, world, dtype):
    Z, Hq, Hkv, L = 2, 4, 2, 3000  # ragged last block, M = 24
    q, k, v = fp.workload.composite(9, Z, Hq, Hkv, L, dtype=dtype, device="cuda")
    cfg = fp.PipelineConfig(alpha=0.12)
    grid = fp.make_block_grid(L, 128)
    tau = 1 / math.sqrt(128)
    M = grid.num_query_blocks
    plan = fp.discover_select(q, k, cfg)[0]
    whole = fp.block_sparse_attention(q, k, v, plan, grid, tau, out_dtype=torch.float32)
    seen = torch.zeros(M, dtype=torch.bool)
    for rank in range(world):
        rows = (rank, world)
        pr = fp.discover_select(q, k, cfg, rows=rows)[0]
        own = list(range(rank, M, world))
        seen[own] = True
        assert torch.equal(pr.counts[:, own], plan.counts[:, own])
        for I in own:  # live slots of each owned plan row (fill value N beyond the count)
            assert torch.equal(pr.indices[:, I], plan.indices[:, I])
        res = fp.block_sparse_attention(q, k, v, pr, grid, tau, out_dtype=torch.float32,
                                        rows=rows)
        for I in own:
            sl = slice(I * 128, min(L, (I + 1) * 128))
            assert torch.equal(res.out[:, :, sl], whole.out[:, :, sl])
            assert torch.equal(res.lse[:, :, sl], whole.lse[:, :, sl])
    assert bool(seen.all())


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_zigzag_shards_equal_whole(fp, world):
    """Zigzag shards (fpb_*_zigzag: chunks rank and 2G-1-rank of 2G contiguous chunks) produce
    exactly the unsharded plan rows and output rows, and together cover every query block; world 8
    at M = 24 leaves some ranks' high chunk partly or wholly beyond the last block."""
    Z, Hq, Hkv, L = 2, 4, 2, 3000  # ragged last block, M = 24
    q, k, v = fp.workload.composite(9, Z, Hq, Hkv, L, device="cuda")
    cfg = fp.PipelineConfig(alpha=0.12)
    grid = fp.make_block_grid(L, 128)
    tau = 1 / math.sqrt(128)
    M = grid.num_query_blocks
    plan = fp.discover_select(q, k, cfg)[0]
    whole = fp.block_sparse_attention(q, k, v, plan, grid, tau, out_dtype=torch.float32)
    seen = torch.zeros(M, dtype=torch.int32)
    for rank in range(world):
        rows = fp.shard.zigzag_shard(world, rank)
        own = fp.shard.zigzag_blocks(M, world, rank)
        seen[own] += 1
        pr = fp.discover_select(q, k, cfg, rows=rows)[0]
        assert torch.equal(pr.counts[:, own], plan.counts[:, own])
        for I in own:
            assert torch.equal(pr.indices[:, I], plan.indices[:, I])
        res = fp.block_sparse_attention(q, k, v, pr, grid, tau, out_dtype=torch.float32,
                                        rows=rows)
        for I in own:
            sl = slice(I * 128, min(L, (I + 1) * 128))
            assert torch.equal(res.out[:, :, sl], whole.out[:, :, sl])
            assert torch.equal(res.lse[:, :, sl], whole.lse[:, :, sl])
    assert bool((seen == 1).all())


@pytest.mark.parametrize("part", ["rows", "zigzag"])
def test_long_row_shards_fill_owned_rows(fp, part):
    """M >= 1024 key blocks: the plan rows are prefilled with N by fill_plan_kernel and the fused
    epilogue then writes only the active slots.  The prefill must hit exactly the rank's owned rows
    (interleaved or zigzag), so every owned row -- fill slots included -- equals the unsharded
    plan row (selection.hpp:176-192: slots >= C hold N)."""
    Z, Hq, Hkv, L = 1, 2, 1, 1030 * 128 - 5  # M = 1030, ragged last block
    q, k, _ = fp.workload.composite(21, Z, Hq, Hkv, L, device="cuda")
    cfg = fp.PipelineConfig(alpha=0.12)
    M = fp.make_block_grid(L, 128).num_query_blocks
    plan = fp.discover_select(q, k, cfg)[0]
    world = 3
    for rank in range(world):
        if part == "rows":
            rows, own = (rank, world), list(range(rank, M, world))
        else:
            rows, own = fp.shard.zigzag_shard(world, rank), fp.shard.zigzag_blocks(M, world, rank)
        pr = fp.discover_select(q, k, cfg, rows=rows)[0]
        own_t = torch.as_tensor(own, device="cuda")
        assert torch.equal(pr.counts[:, own_t], plan.counts[:, own_t]), (part, rank)
        assert torch.equal(pr.indices[:, own_t], plan.indices[:, own_t]), (part, rank)


def test_zigzag_runner_and_validation(fp):
    """PrefillRunner graphs on a zigzag shard reproduce the direct calls; rank outside
    [0, world) is a ValidationError."""
    Z, Hq, Hkv, L = 1, 4, 2, 2000
    q, k, v = fp.workload.composite(4, Z, Hq, Hkv, L, device="cuda")
    cfg = fp.PipelineConfig(alpha=0.1)
    grid = fp.make_block_grid(L, 128)
    M = grid.num_query_blocks
    plan = fp.discover_select(q, k, cfg)[0]
    ref = fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128),
                                    out_dtype=torch.bfloat16)
    rows = fp.shard.zigzag_shard(3, 1)
    r = fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16, rows=rows).capture()
    r.replay_discover()
    r.replay_attend()
    r.check()
    for I in fp.shard.zigzag_blocks(M, 3, 1):
        sl = slice(I * 128, min(L, (I + 1) * 128))
        assert torch.equal(r.out[:, :, sl], ref.out[:, :, sl])
    with pytest.raises(fp.ValidationError):
        fp.discover_select(q, k, cfg, rows=("zigzag", 3, 3))


def test_row_shard_beyond_blocks_is_noop(fp):
    """A rank whose row_begin is past the last block owns nothing: both calls return without
    touching their outputs."""
    L = 256  # M = 2 blocks, rank 5 of 8 owns none
    q, k, v = fp.workload.composite(1, 1, 2, 1, L, device="cuda")
    cfg = fp.PipelineConfig()
    plan = fp.discover_select(q, k, cfg)[0]
    grid = fp.make_block_grid(L, 128)
    pr = fp.discover_select(q, k, cfg, rows=(5, 8))[0]
    assert pr.counts.shape == plan.counts.shape
    fp.block_sparse_attention(q, k, v, plan, grid, 1 / math.sqrt(128), rows=(5, 8))


def test_row_shard_validation(fp):
    q, k, v = fp.workload.composite(1, 1, 2, 1, 512, device="cuda")
    with pytest.raises(fp.ValidationError):
        fp.discover_select(q, k, fp.PipelineConfig(), rows=(2, 2))
    with pytest.raises(fp.ValidationError):
        fp.discover_select(q, k, fp.PipelineConfig(), rows=(0, 0))


@pytest.mark.parametrize("rows", [None, (1, 2)])
def test_prefill_runner_graph_replay(fp, rows):
    """PrefillRunner (preallocated buffers, two CUDA graphs) reproduces the direct calls."""
    Z, Hq, Hkv, L = 1, 4, 2, 2000
    q, k, v = fp.workload.composite(4, Z, Hq, Hkv, L, device="cuda")
    cfg = fp.PipelineConfig(alpha=0.1)
    grid = fp.make_block_grid(L, 128)
    plan = fp.discover_select(q, k, cfg)[0]
    ref = fp.block_sparse_attention(q, k, v, plan, grid, cfg.resolved_scale(128),
                                    out_dtype=torch.bfloat16)
    r = fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16, rows=rows).capture()
    for _ in range(3):
        r.replay_discover()
        r.replay_attend()
    visits = r.check()
    M = grid.num_query_blocks
    own = list(range(M)) if rows is None else list(range(rows[0], M, rows[1]))
    assert torch.equal(r.counts[:, own], plan.counts[:, own])
    for I in own:
        sl = slice(I * 128, min(L, (I + 1) * 128))
        assert torch.equal(r.out[:, :, sl], ref.out[:, :, sl])
        assert torch.equal(r.lse[:, :, sl], ref.lse[:, :, sl])
    # 1 warm-up launch + 3 replays, visits accumulate per launch
    assert visits == 4 * int(plan.counts[:, own].to(torch.int64).sum())


def test_one_million_tokens_single_head(fp):
    """Maximum-size case: L = 2^20 tokens (M = 8192 key blocks, per-key-block rows in the global
    scratch, plan 256 MiB), one Q / KV head.  Plan invariants of the reference
    (selection.hpp:176-192) and two full query blocks of the output recomputed in float64 from
    the plan (attention.hpp:38-132)."""
    import numpy as np
    L = 1 << 20
    q, k, v = fp.workload.composite(17, 1, 1, 1, L, device="cuda")
    cfg = fp.PipelineConfig(alpha=0.12)
    grid = fp.make_block_grid(L, 128)
    tau = cfg.resolved_scale(128)
    plan = fp.discover_select(q, k, cfg)[0]
    M = grid.num_query_blocks
    cnt = plan.counts[0, :, 0]
    assert bool((cnt >= 1).all()) and bool((cnt <= torch.arange(M, device="cuda") + 1).all())
    res = fp.block_sparse_attention(q, k, v, plan, grid, tau, out_dtype=torch.float32)
    assert bool(torch.isfinite(res.out).all()) and bool(torch.isfinite(res.lse).all())
    for I in (M // 3, M - 1):
        c = int(cnt[I])
        blocks = plan.indices[0, I, :c, 0].cpu().numpy()
        assert np.all(np.diff(blocks) > 0) and blocks[0] == 0 and blocks[-1] == I
        qi = q[0, 0, I * 128:(I + 1) * 128].double().cpu().numpy()
        keys = np.concatenate([np.arange(j * 128, (j + 1) * 128) for j in blocks])
        kk = k[0, 0].double().cpu().numpy()[keys]
        vv = v[0, 0].double().cpu().numpy()[keys]
        x = (qi @ kk.T) * tau * np.log2(np.e)
        rows = np.arange(I * 128, (I + 1) * 128)[:, None]
        x[keys[None, :] > rows] = -np.inf  # causal mask inside the diagonal block only
        m = x.max(axis=1, keepdims=True)
        p = np.exp2(x - m)
        o = (p @ vv) / p.sum(axis=1, keepdims=True)
        lse = m[:, 0] + np.log2(p.sum(axis=1))
        go = res.out[0, 0, I * 128:(I + 1) * 128].double().cpu().numpy()
        gl = res.lse[0, 0, I * 128:(I + 1) * 128].double().cpu().numpy()
        assert np.abs(go - o).max() <= 2e-2 and np.abs(go - o).mean() <= 1e-3
        assert np.abs(gl - lse).max() <= 2e-2
