"""world_size-2 gloo test of the N>1 host path: each rank computes its KV-head-group shard of the
prefill (CPU oracle standing in for the per-rank kernels) and the head all-gather reassembles the
full output, equal to the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, k, v, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from paper_2603_06199_b200.shard import gather_heads, kv_group_shard, local_slices
    o = Oracle("port")
    Hq, Hkv = q.shape[1], k.shape[1]
    s = kv_group_shard(Hq, Hkv, world, rank)
    ql, kl, vl = (x.numpy() for x in local_slices(q, k, v, s))
    tau = float(o.scale(ql.shape[-1]))
    _, _, sc = o.discover(ql, kl, 128, tau)
    mask, _ = o.max_threshold_mask(sc, 128, 0.12, 256, 512)
    idx, counts = o.compress_indices(mask)
    out, lse, _ = o.block_sparse_attention(ql, kl, vl, idx, counts, 128, tau)
    full_o, full_l = gather_heads(torch.from_numpy(out), torch.from_numpy(lse), Hq, Hkv)
    if rank == 0:
        ret["out"] = full_o.numpy()
        ret["lse"] = full_l.numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather():
    from oracle import Oracle
    from tests._util import composite_np
    Z, Hq, Hkv, L = 1, 4, 2, 512
    q, k, v = (torch.from_numpy(x) for x in composite_np(3, Z, Hq, Hkv, L))
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), q, k, v, ret), nprocs=world, join=True)
    o = Oracle("port")
    qn, kn, vn = q.numpy(), k.numpy(), v.numpy()
    tau = float(o.scale(128))
    _, _, sc = o.discover(qn, kn, 128, tau)
    mask, _ = o.max_threshold_mask(sc, 128, 0.12, 256, 512)
    idx, counts = o.compress_indices(mask)
    out, lse, _ = o.block_sparse_attention(qn, kn, vn, idx, counts, 128, tau)
    assert np.array_equal(ret["out"], out) and np.array_equal(ret["lse"], lse)


def _rows_worker(rank, world, port, out, lse, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_06199_b200.shard import gather_rows, row_shard
    rb, rs = row_shard(world, rank)
    L = out.shape[2]
    own = torch.zeros(L, dtype=torch.bool)
    for I in range(rb, -(-L // 128), rs):
        own[I * 128:(I + 1) * 128] = True
    # rows this rank does not own are garbage in its buffers (fpb_*_rows leaves them unwritten)
    o = torch.where(own[None, None, :, None], out, torch.full_like(out, float("nan")))
    l_ = torch.where(own[None, None, :], lse, torch.full_like(lse, -7.0))
    go, gl = gather_rows(o, l_, 128)
    if rank == 0:
        ret["out"] = go.numpy()
        ret["lse"] = gl.numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_row_shard_gather_ragged_three_ranks():
    """Row-sharded partition (query blocks r, r + G, ... per rank): the all-gather reassembles
    the full output, including a ragged last block and M not divisible by the world size."""
    g = torch.Generator().manual_seed(0)
    Z, Hq, L, d = 2, 3, 1000, 128  # M = 8 blocks over 3 ranks
    out = torch.randn((Z, Hq, L, d), generator=g)
    lse = torch.randn((Z, Hq, L), generator=g)
    world = 3
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_rows_worker, args=(world, _free_port(), out, lse, ret), nprocs=world, join=True)
    assert np.array_equal(ret["out"], out.numpy()) and np.array_equal(ret["lse"], lse.numpy())


def _zigzag_worker(rank, world, port, out, lse, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_06199_b200.shard import gather_zigzag, zigzag_blocks
    L = out.shape[2]
    own = torch.zeros(L, dtype=torch.bool)
    for I in zigzag_blocks(-(-L // 128), world, rank):
        own[I * 128:(I + 1) * 128] = True
    # rows this rank does not own are garbage in its buffers (fpb_*_zigzag leaves them unwritten)
    o = torch.where(own[None, None, :, None], out, torch.full_like(out, float("nan")))
    l_ = torch.where(own[None, None, :], lse, torch.full_like(lse, -7.0))
    go, gl = gather_zigzag(o, l_, 128)
    if rank == 0:
        ret["out"] = go.numpy()
        ret["lse"] = gl.numpy()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 1000), (3, 1300)])
def test_zigzag_shard_gather(world, L):
    """Zigzag partition (two contiguous chunks per rank): the all-gather reassembles the full
    output, including a ragged last block and a chunk grid that does not divide M."""
    g = torch.Generator().manual_seed(world)
    Z, Hq, d = 2, 3, 128
    out = torch.randn((Z, Hq, L, d), generator=g)
    lse = torch.randn((Z, Hq, L), generator=g)
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_zigzag_worker, args=(world, _free_port(), out, lse, ret), nprocs=world, join=True)
    assert np.array_equal(ret["out"], out.numpy()) and np.array_equal(ret["lse"], lse.numpy())


@pytest.mark.parametrize("M", [1, 5, 16, 17, 100, 2048])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_zigzag_blocks_partition(M, world):
    """Every query block is owned by exactly one rank; each rank owns at most two contiguous
    chunks of ceil(M / 2 world) blocks."""
    from paper_2603_06199_b200.shard import zigzag_blocks
    owned = [zigzag_blocks(M, world, r) for r in range(world)]
    assert sorted(b for o in owned for b in o) == list(range(M))
    c = -(-M // (2 * world))
    assert all(len(o) <= 2 * c for o in owned)


def _overlap_worker(rank, world, port, Hq, Hkv, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_06199_b200 import shard
    L, d = 40, 8
    full = torch.arange(Hq * L * d, dtype=torch.float32).view(1, Hq, L, d)
    full_l = -torch.arange(Hq * L, dtype=torch.float32).view(1, Hq, L)
    s = shard.kv_group_shard(Hq, Hkv, world, rank)
    out, lse = torch.zeros_like(full), torch.zeros_like(full_l)
    g = shard.OverlappedHeadGather(Hq, Hkv, out, lse)
    for a, b in shard.head_chunks(s.hq, 2):  # bench.py's chunked KV step: P2P per head chunk
        g.post(a, b, full[:, s.q_lo + a:s.q_lo + b], full_l[:, s.q_lo + a:s.q_lo + b])
    g.wait()
    ret[rank] = bool(torch.equal(out, full) and torch.equal(lse, full_l))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,Hq,Hkv", [(2, 8, 2), (4, 8, 2), (4, 12, 2), (3, 6, 3)])
def test_overlapped_head_gather(world, Hq, Hkv):
    """shard.OverlappedHeadGather (the chunked P2P gather bench.py overlaps with compute) puts
    every rank's head chunks at their place in the full layer, on every rank."""
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_overlap_worker, args=(world, _free_port(), Hq, Hkv, ret), nprocs=world, join=True)
    assert all(ret[r] for r in range(world)), dict(ret)


def test_head_chunks():
    from paper_2603_06199_b200.shard import head_chunks
    assert head_chunks(4, 2) == [(0, 2), (2, 4)]
    assert head_chunks(3, 2) == [(0, 2), (2, 3)]
    assert head_chunks(1, 4) == [(0, 1)]
    assert head_chunks(16, 3) == [(0, 6), (6, 11), (11, 16)]


def _kvz_worker(rank, world, port, Hkv, out, lse, ret, weights=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_06199_b200.shard import gather_kv_zigzag, kv_zigzag_shard, zigzag_blocks
    Hq, L = out.shape[1], out.shape[2]
    s, rows = kv_zigzag_shard(Hq, Hkv, world, rank, weights)
    own = torch.zeros(L, dtype=torch.bool)
    blocks = range(-(-L // 128)) if rows is None else zigzag_blocks(-(-L // 128), rows[2], rows[1])
    for I in blocks:
        own[I * 128:(I + 1) * 128] = True
    # the rank's KV group; rows it does not own are garbage (fpb_*_zigzag leaves them unwritten)
    o = out[:, s.q_lo:s.q_hi].clone()
    l_ = lse[:, s.q_lo:s.q_hi].clone()
    o[:, :, ~own] = float("nan")
    l_[:, :, ~own] = -7.0
    go, gl = gather_kv_zigzag(o, l_, Hq, Hkv, 128, weights=weights)
    ret[rank] = bool(torch.equal(go, out) and torch.equal(gl, lse))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,Hq,Hkv,L,weights", [
    (2, 4, 1, 1000, None), (4, 8, 2, 1300, None), (4, 4, 4, 700, None), (3, 6, 1, 2000, None),
    (8, 16, 4, 1500, (20.1, 10.9, 6.2, 16.3)),  # ranks per group 3, 2, 1, 2
    (4, 8, 4, 900, (1.0, 1.0, 1.0, 1.0))])      # weighted, one rank per group
def test_kv_zigzag_gather(world, Hq, Hkv, L, weights):
    """kv_zigzag partition: one KV group per rank (or per world/Hkv ranks, each with all of the
    group's Q heads and its zigzag chunks); the gather reassembles the full layer on every rank,
    ragged last block included."""
    g = torch.Generator().manual_seed(world * 31 + L)
    out = torch.randn((1, Hq, L, 128), generator=g)
    lse = torch.randn((1, Hq, L), generator=g)
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_kvz_worker, args=(world, _free_port(), Hkv, out, lse, ret, weights), nprocs=world,
             join=True)
    assert all(ret[r] for r in range(world)), dict(ret)


@pytest.mark.parametrize("world,Hq,Hkv,weights", [
    (1, 8, 2, None), (2, 8, 2, None), (4, 8, 2, None), (8, 32, 4, None), (3, 6, 1, None),
    (8, 32, 4, (20.1, 10.9, 6.2, 16.3)), (7, 32, 4, (1, 5, 1, 1)), (4, 8, 4, (3, 1, 2, 2))])
def test_kv_zigzag_shard_covers_layer(world, Hq, Hkv, weights):
    """Every (Q head, query block) is owned by exactly one rank; a rank holds one KV head's group
    (or whole groups when world <= Hkv)."""
    from paper_2603_06199_b200.shard import kv_zigzag_shard, zigzag_blocks
    M = 37
    seen = {}
    for r in range(world):
        s, rows = kv_zigzag_shard(Hq, Hkv, world, r, weights)
        assert s.q_hi - s.q_lo == (s.kv_hi - s.kv_lo) * (Hq // Hkv)
        blocks = range(M) if rows is None else zigzag_blocks(M, rows[2], rows[1])
        for h in range(s.q_lo, s.q_hi):
            for I in blocks:
                assert (h, I) not in seen
                seen[(h, I)] = r
    assert len(seen) == Hq * M


def test_kv_group_ranks_by_weight():
    """Heavier KV groups get more ranks; every group at least one; equal split without weights."""
    from paper_2603_06199_b200.shard import kv_group_ranks
    assert kv_group_ranks(4, 8) == [2, 2, 2, 2]
    assert kv_group_ranks(4, 8, [20.1, 10.9, 6.2, 16.3]) == [3, 2, 1, 2]
    assert kv_group_ranks(4, 4, [9, 1, 1, 1]) == [1, 1, 1, 1]
    assert sum(kv_group_ranks(8, 13, list(range(1, 9)))) == 13
    with pytest.raises(ValueError):
        kv_group_ranks(4, 6)  # equal split needs divisibility
