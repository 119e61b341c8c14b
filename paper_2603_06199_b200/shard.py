"""Multi-GPU partitioning of the FlashPrefill path.

Every (z, Q head) is independent through discovery, selection and attention
(discovery.hpp:87-88, selection.hpp:71-72, attention.hpp:59-60), so the path shards with no
data-path collective:

* ``kv_group_shard`` — strong scaling of one batch by KV-head groups: rank g owns KV heads
  [g*Hkv/G, (g+1)*Hkv/G) and their Q heads; with G > Hkv each group's Q heads are split over
  G/Hkv ranks and the KV head is replicated (e.g. Qwen3 Hkv=4 on 8 GPUs: 4 Q heads per rank).
* ``kv_zigzag_shard`` — the same KV-head groups, but with more ranks than KV heads a group is
  split by zigzag query-block chunks (all of its Q heads on every rank of the group) instead of by
  Q heads, so the ranks of a group carry equal work whatever the per-head densities
  (``gather_kv_zigzag`` reassembles it).
* ``unit_shard`` — weak scaling: work units (sequence, KV-head group) dealt contiguously.
* ``gather_heads`` — the only collective: one all-gather of O and LSE along the head axis after
  all kernels complete (NCCL over NVLink in production, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class HeadShard:
    q_lo: int
    q_hi: int
    kv_lo: int
    kv_hi: int

    @property
    def hq(self) -> int:
        return self.q_hi - self.q_lo

    @property
    def hkv(self) -> int:
        return self.kv_hi - self.kv_lo


def kv_group_shard(Hq: int, Hkv: int, world: int, rank: int) -> HeadShard:
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    g = Hq // Hkv
    if world <= Hkv:
        if Hkv % world:
            raise ValueError(f"{world} ranks do not divide {Hkv} KV heads")
        per = Hkv // world
        return HeadShard(rank * per * g, (rank + 1) * per * g, rank * per, (rank + 1) * per)
    if world % Hkv or g % (world // Hkv):
        raise ValueError(f"{world} ranks cannot split {Hkv} KV groups of {g} Q heads")
    split = world // Hkv  # ranks per KV group
    kv = rank // split
    per_q = g // split
    q0 = kv * g + (rank % split) * per_q
    return HeadShard(q0, q0 + per_q, kv, kv + 1)


def kv_group_ranks(Hkv: int, world: int, weights=None) -> list[int]:
    """Ranks per KV group for world >= Hkv: equal (world / Hkv each) without weights; with
    per-group work weights (e.g. the plan's block visits per KV group from a calibration pass),
    every group gets one rank and each further rank goes to the group with the largest work per
    rank, so heavy groups are split over more ranks (profiles/r2_kv_zigzag.md)."""
    if world < Hkv:
        raise ValueError("fewer ranks than KV groups: use kv_group_shard")
    if weights is None:
        if world % Hkv:
            raise ValueError(f"{world} ranks cannot split {Hkv} KV groups evenly")
        return [world // Hkv] * Hkv
    if len(weights) != Hkv:
        raise ValueError("one weight per KV group")
    n = [1] * Hkv
    for _ in range(world - Hkv):
        g = max(range(Hkv), key=lambda i: (weights[i] / n[i], -i))
        n[g] += 1
    return n


def kv_zigzag_shard(Hq: int, Hkv: int, world: int, rank: int, weights=None):
    """KV-head-group shard that splits a group by query rows instead of Q heads.

    Returns (HeadShard, rows): with world <= Hkv (and no weights) it is kv_group_shard and rows is
    None; otherwise the ranks of a KV group (kv_group_ranks: equal, or by work weights) each take
    ALL of the group's Q heads but only the zigzag query-block chunks (sub, 2 n - 1 - sub) of an
    n-rank zigzag partition (rows = ("zigzag", sub, n), fpb_*_zigzag).  A rank still holds exactly
    one KV head (the north_star partition), but its work no longer depends on which Q heads it
    drew: per-head densities differ several-fold (profiles/r2_lsweep.md)."""
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    if world <= Hkv and (weights is None or world < Hkv):
        return kv_group_shard(Hq, Hkv, world, rank), None
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    n = kv_group_ranks(Hkv, world, weights)
    g = Hq // Hkv
    kv, first = 0, 0
    while rank >= first + n[kv]:
        first += n[kv]
        kv += 1
    rows = ("zigzag", rank - first, n[kv]) if n[kv] > 1 else None
    return HeadShard(kv * g, (kv + 1) * g, kv, kv + 1), rows


def unit_shard(n_units: int, world: int, rank: int) -> range:
    per, extra = divmod(n_units, world)
    lo = rank * per + min(rank, extra)
    return range(lo, lo + per + (1 if rank < extra else 0))


def local_slices(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, s: HeadShard):
    """Contiguous per-rank head slices of Z x H x L x d tensors."""
    return (q[:, s.q_lo:s.q_hi].contiguous(), k[:, s.kv_lo:s.kv_hi].contiguous(),
            v[:, s.kv_lo:s.kv_hi].contiguous())


def _all_gather(dst: torch.Tensor, src: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor; over gloo (CPU tests, the shared-GPU test mode) device tensors
    are staged through host memory."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    src = src.reshape(1, -1)  # rank-major chunks along dim 0 (gloo requires it)
    if dist.get_backend(group) == "gloo" and src.is_cuda:
        tmp = torch.empty((world, src.shape[1]), dtype=dst.dtype)
        dist.all_gather_into_tensor(tmp, src.cpu(), group=group)
        dst.copy_(tmp.view(dst.shape))
    else:
        dist.all_gather_into_tensor(dst.view(world, -1), src, group=group)


def gather_heads(out_local: torch.Tensor, lse_local: torch.Tensor, Hq: int, Hkv: int,
                 group=None, out: torch.Tensor | None = None, lse: torch.Tensor | None = None):
    """All-gather per-rank (Z x hq_local x L x d, Z x hq_local x L) along the head axis.

    For Z = 1 the ranks' head ranges are contiguous and ascending, so the collective writes the
    final Z x Hq x L x d layout directly (no staging copy); `out` / `lse` may be preallocated."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    Z, hl, L, d = out_local.shape
    if out is None:
        out = torch.empty((Z, Hq, L, d), dtype=out_local.dtype, device=out_local.device)
    if lse is None:
        lse = torch.empty((Z, Hq, L), dtype=lse_local.dtype, device=lse_local.device)
    order = [kv_group_shard(Hq, Hkv, world, r).q_lo for r in range(world)]
    if Z == 1 and order == [r * hl for r in range(world)] and world * hl == Hq:
        _all_gather(out, out_local.contiguous(), group)
        _all_gather(lse, lse_local.contiguous(), group)
        return out, lse
    # head-major staging so one all_gather_into_tensor moves every rank's block contiguously
    ob = torch.empty((world * Z, hl, L, d), dtype=out_local.dtype, device=out_local.device)
    lb = torch.empty((world * Z, hl, L), dtype=lse_local.dtype, device=lse_local.device)
    _all_gather(ob, out_local.contiguous(), group)
    _all_gather(lb, lse_local.contiguous(), group)
    ob, lb = ob.view(world, Z, hl, L, d), lb.view(world, Z, hl, L)
    for r, q0 in enumerate(order):
        out[:, q0:q0 + hl] = ob[r]
        lse[:, q0:q0 + hl] = lb[r]
    return out, lse


def head_chunks(hl: int, chunks: int) -> list[tuple[int, int]]:
    """A rank's hl local Q heads as `chunks` contiguous ranges (sizes differ by at most one)."""
    chunks = max(1, min(chunks, hl))
    per, extra = divmod(hl, chunks)
    out, lo = [], 0
    for c in range(chunks):
        hi = lo + per + (1 if c < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class OverlappedHeadGather:
    """The O / LSE all-gather of a KV-group-sharded layer (Z = 1), posted chunk by chunk so it
    runs on the collective stream while the rank computes its next chunk of Q heads.

    Every rank owns the same number of Q heads (kv_group_shard), split the same way into chunks, so
    chunk c of rank p lands at heads [q_lo(p) + a_c, q_lo(p) + b_c) of the full layer.  post(c, ...)
    sends this rank's chunk to every peer and receives every peer's chunk straight into `out` /
    `lse` with point-to-point operations (one NCCL group: no staging buffer, no permuting copy);
    wait() makes the current stream wait for everything posted.  Over gloo (the CPU tests and the
    shared-GPU test mode) the transfers are staged through host memory and complete in post()."""

    def __init__(self, Hq: int, Hkv: int, out: torch.Tensor, lse: torch.Tensor, group=None):
        import torch.distributed as dist
        if out.shape[0] != 1:
            raise ValueError("the overlapped gather needs Z = 1 (heads contiguous per rank)")
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.q_lo = [kv_group_shard(Hq, Hkv, self.world, r).q_lo for r in range(self.world)]
        self.out, self.lse = out, lse
        self.gloo = dist.get_backend(group) == "gloo"
        self.works = []

    def post(self, lo: int, hi: int, out_c: torch.Tensor, lse_c: torch.Tensor) -> None:
        """This rank's local heads [lo, hi) (out_c: 1 x (hi-lo) x L x d, lse_c: 1 x (hi-lo) x L)."""
        d = self.dist
        me = self.q_lo[self.rank]
        self.out[:, me + lo:me + hi].copy_(out_c)
        self.lse[:, me + lo:me + hi].copy_(lse_c)
        peers = [p for p in range(self.world) if p != self.rank]
        if self.gloo:  # host-staged, synchronous
            src_o, src_l = out_c.contiguous().cpu(), lse_c.contiguous().cpu()
            for step in range(1, self.world):  # pairwise exchange, deadlock-free ring order
                to, frm = (self.rank + step) % self.world, (self.rank - step) % self.world
                ro = torch.empty_like(src_o)
                rl = torch.empty_like(src_l)
                ops = [d.P2POp(d.isend, src_o, to, self.group), d.P2POp(d.irecv, ro, frm, self.group),
                       d.P2POp(d.isend, src_l, to, self.group), d.P2POp(d.irecv, rl, frm, self.group)]
                for w in d.batch_isend_irecv(ops):
                    w.wait()
                q0 = self.q_lo[frm]
                self.out[:, q0 + lo:q0 + hi].copy_(ro)
                self.lse[:, q0 + lo:q0 + hi].copy_(rl)
            return
        ops = []
        src_o, src_l = out_c.contiguous(), lse_c.contiguous()
        for p in peers:
            q0 = self.q_lo[p]
            ops += [d.P2POp(d.isend, src_o, p, self.group),
                    d.P2POp(d.irecv, self.out[:, q0 + lo:q0 + hi], p, self.group),
                    d.P2POp(d.isend, src_l, p, self.group),
                    d.P2POp(d.irecv, self.lse[:, q0 + lo:q0 + hi], p, self.group)]
        self.works += d.batch_isend_irecv(ops)

    def wait(self) -> None:
        for w in self.works:
            w.wait()
        self.works = []


# ----------------------------------------------------------------------------- row sharding
# Strong scaling without the KV-group imbalance: rank r of G owns query blocks r, r + G, ...
# of EVERY head (fpb_discover_select_rows / fpb_block_sparse_attention_rows with
# row_begin = r, row_step = G).  Per-head densities differ a lot (the planted patterns, and real
# heads), so KV-group shards finish at very different times (max/mean 1.8 at Qwen3 256K on 8
# ranks, profiles/r1_lsweep.md); interleaved query blocks give every rank the same mix of heads
# and row lengths.  Cost: every rank holds the whole K/V (2 x L x Hkv x d bf16: 512 MiB at 256K
# Qwen3, trivial next to 180 GB of HBM) and pools all key blocks itself (~0.06 ms).

def row_shard(world: int, rank: int) -> tuple[int, int]:
    """(row_begin, row_step) of rank `rank` out of `world`."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank, world


def zigzag_shard(world: int, rank: int) -> tuple[str, int, int]:
    """Rank's zigzag shard (fpb_*_zigzag): query blocks cut into 2 * world contiguous chunks of
    ceil(M / (2 world)); rank owns chunks rank and 2 world - 1 - rank (equal causal work,
    contiguous rows)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return ("zigzag", rank, world)


def zigzag_blocks(M: int, world: int, rank: int) -> list[int]:
    """The query blocks a zigzag shard owns (ascending); mirrors restrict_zigzag in csrc/abi.cu."""
    c = -(-M // (2 * world))
    lo = range(rank * c, min(M, (rank + 1) * c))
    hi = range((2 * world - 1 - rank) * c, min(M, (2 * world - rank) * c))
    return list(lo) + list(hi)


def gather_zigzag(out: torch.Tensor, lse: torch.Tensor, block: int, group=None):
    """All-gather a zigzag-sharded result (every rank holds full-size out / lse with only its two
    chunks written); returns the assembled tensors."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    res = []
    for x in (out, lse):
        Z, H, L = x.shape[:3]
        M = -(-L // block)
        c = -(-M // (2 * world))
        Lp = 2 * world * c * block
        if Lp != L:
            pad = torch.zeros((Z, H, Lp) + tuple(x.shape[3:]), dtype=x.dtype, device=x.device)
            pad[:, :, :L] = x
            x = pad
        xc = x.view((Z, H, 2 * world, c * block) + tuple(x.shape[3:]))
        mine = torch.stack((xc[:, :, rank], xc[:, :, 2 * world - 1 - rank]), dim=2).contiguous()
        allr = torch.empty((world * Z,) + tuple(mine.shape[1:]), dtype=x.dtype, device=x.device)
        _all_gather(allr, mine, group)
        allr = allr.view((world,) + tuple(mine.shape))  # rank, Z, H, 2, cB, ...
        chunks = [allr[r, :, :, 0] for r in range(world)] + \
                 [allr[r, :, :, 1] for r in reversed(range(world))]
        full = torch.stack(chunks, dim=2).reshape((Z, H, Lp) + tuple(x.shape[3:]))[:, :, :L]
        res.append(full.contiguous())
    return res[0], res[1]


def _row_blocks(x: torch.Tensor, block: int, world: int):
    """Pad the L axis (dim 2) to a multiple of block * world and expose (.., M/world, world, B, ..)."""
    Z, H, L = x.shape[:3]
    M = -(-L // block)
    Mw = -(-M // world) * world
    if Mw * block != L:
        pad = torch.zeros((Z, H, Mw * block) + tuple(x.shape[3:]), dtype=x.dtype, device=x.device)
        pad[:, :, :L] = x
        x = pad
    return x.view((Z, H, Mw // world, world, block) + tuple(x.shape[3:])), L


def gather_rows(out: torch.Tensor, lse: torch.Tensor, block: int, group=None):
    """All-gather a row-sharded result.  Every rank holds full-size out (Z x Hq x L x d) and lse
    (Z x Hq x L) with only its own query blocks written; returns the assembled tensors."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    res = []
    for x in (out, lse):
        xb, L = _row_blocks(x, block, world)
        mine = xb[:, :, :, rank].contiguous()
        allr = torch.empty((world * mine.shape[0],) + tuple(mine.shape[1:]), dtype=x.dtype,
                           device=x.device)
        _all_gather(allr, mine, group)
        full = allr.view((world,) + tuple(mine.shape)).movedim(0, 3).contiguous()
        full = full.view((x.shape[0], x.shape[1], -1) + tuple(x.shape[3:]))[:, :, :L]
        res.append(full.contiguous())
    return res[0], res[1]


def gather_kv_zigzag(out_local: torch.Tensor, lse_local: torch.Tensor, Hq: int, Hkv: int,
                     block: int, group=None, out: torch.Tensor | None = None,
                     lse: torch.Tensor | None = None, weights=None):
    """Gather a kv_zigzag_shard result (same Hq, Hkv, weights) on every rank.  out_local /
    lse_local: the rank's KV group (Z x g x L x d, Z x g x L) with only its zigzag chunks written.
    Ranks own differently sized chunks when groups have different rank counts, so every rank
    broadcasts its two chunks (exact sizes) and each lands at (its group's heads, its chunks'
    rows) of the full Z x Hq layout."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world <= Hkv and (weights is None or world < Hkv):
        return gather_heads(out_local, lse_local, Hq, Hkv, group, out, lse)
    rank = dist.get_rank(group)
    g = Hq // Hkv
    Z, _, L = out_local.shape[:3]
    M = -(-L // block)
    spec = []  # per rank: (kv group, [(row lo, row hi) of its two chunks])
    for r in range(world):
        sh, rows = kv_zigzag_shard(Hq, Hkv, world, r, weights)
        if rows is None:
            spec.append((sh.kv_lo, [(0, L), (L, L)]))
            continue
        _, sub, n = rows
        c = -(-M // (2 * n)) * block
        spec.append((sh.kv_lo, [(min(L, ch * c), min(L, (ch + 1) * c))
                                for ch in (sub, 2 * n - 1 - sub)]))
    if out is None:
        out = torch.empty((Z, Hq) + tuple(out_local.shape[2:]), dtype=out_local.dtype,
                          device=out_local.device)
    if lse is None:
        lse = torch.empty((Z, Hq, L), dtype=lse_local.dtype, device=lse_local.device)
    for x, dst in ((out_local, out), (lse_local, lse)):
        tail = tuple(x.shape[3:])
        for r, (kv, chunks) in enumerate(spec):  # one broadcast per rank, exact sizes
            n_rows = sum(b - a for a, b in chunks)
            if r == rank:
                buf = torch.cat([x[:, :, a:b] for a, b in chunks], dim=2).contiguous()
            else:
                buf = torch.empty((Z, g, n_rows) + tail, dtype=x.dtype, device=x.device)
            _broadcast(buf, r, group)
            o = 0
            for a, b in chunks:
                dst[:, kv * g:(kv + 1) * g, a:b] = buf[:, :, o:o + b - a]
                o += b - a
    return out, lse


def _broadcast(t: torch.Tensor, src: int, group=None) -> None:
    """In-place broadcast; over gloo, device tensors are staged through host memory."""
    import torch.distributed as dist
    if dist.get_backend(group) == "gloo" and t.is_cuda:
        h = t.cpu()
        dist.broadcast(h, dist.get_global_rank(group, src) if group else src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, dist.get_global_rank(group, src) if group else src, group=group)


def prefill_sharded(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, config, partition: str = "kv",
                    group=None, weights=None, out_dtype: torch.dtype | None = None):
    """One layer's FlashPrefill step split over the ranks of `group` (one process per GPU), the
    full O / LSE assembled on every rank.  Every rank passes the whole layer (Z x Hq x L x d Q,
    Z x Hkv x L x d K / V, on its own device); it computes only its share:

      "kv"        kv_group_shard  — KV-head groups, a group's Q heads split (north_star)
      "kv_zigzag" kv_zigzag_shard — KV-head groups, a group's query blocks split (zigzag); with
                  `weights` (work per KV group, e.g. a calibration plan's visits) heavier groups
                  get more ranks
      "rows" / "zigzag" — every head's query blocks interleaved / in zigzag chunks

    Returns (out, lse).  Bit-identical to the unsharded call: every (z, h, query block) is
    computed independently (discovery.hpp:87-88, selection.hpp:71-72, attention.hpp:59-60)."""
    import torch.distributed as dist
    from . import bsattn as fp
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    Z, Hq, L, d = q.shape
    Hkv = k.shape[1]
    grid = fp.make_block_grid(L, config.block_size)
    tau = config.resolved_scale(d)

    def run(ql, kl, vl, rows):
        plan, _, _ = fp.discover_select(ql, kl, config, rows=rows)
        return fp.block_sparse_attention(ql, kl, vl, plan, grid, tau, out_dtype=out_dtype,
                                         rows=rows)

    if world == 1:
        res = run(q, k, v, None)
        return res.out, res.lse
    if partition == "kv":
        s = kv_group_shard(Hq, Hkv, world, rank)
        res = run(*local_slices(q, k, v, s), None)
        return gather_heads(res.out, res.lse, Hq, Hkv, group)
    if partition == "kv_zigzag":
        s, rows = kv_zigzag_shard(Hq, Hkv, world, rank, weights)
        res = run(*local_slices(q, k, v, s), rows)
        return gather_kv_zigzag(res.out, res.lse, Hq, Hkv, config.block_size, group,
                                weights=weights)
    if partition == "rows":
        res = run(q, k, v, row_shard(world, rank))
        return gather_rows(res.out, res.lse, config.block_size, group)
    if partition == "zigzag":
        res = run(q, k, v, zigzag_shard(world, rank))
        return gather_zigzag(res.out, res.lse, config.block_size, group)
    raise ValueError(f"unknown partition {partition!r}")
