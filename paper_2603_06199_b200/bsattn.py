"""Host-side mirror of the reference's ``bsattn::`` API over the sm_100a kernels.

Same names, argument meaning, layouts and error behaviour as /root/reference/proj/include/bsattn/
(core.hpp, discovery.hpp, selection.hpp, attention.hpp), with tensors living in HBM as torch CUDA
tensors (Z x H x L x d, bf16 or fp32).  Every compute call goes through the C ABI of
libfpb200.so (include/fpb200.h); torch only allocates device memory and supplies the stream.
There is no CPU fallback: a missing library or a non-CUDA tensor raises.

GQA (not in the reference): K/V may carry Hkv heads with Hkv | Hq; maps and plans are
per Q head and Q head h reads KV head h // (Hq // Hkv).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import torch

from . import _abi

# ----------------------------------------------------------------------------- errors
# tensor.hpp:18-38


class IoError(RuntimeError):
    pass


class FormatError(RuntimeError):
    pass


class ValidationError(RuntimeError):
    pass


class ConfigError(ValidationError):
    pass


class PlanError(ValidationError):
    pass


class CudaError(RuntimeError):
    pass


def _raise(rc: int, what: str, plan: bool = False):
    if rc == _abi.FPB_OK:
        return
    msg = f"{what}: {_abi.last_error()}"
    if rc == _abi.FPB_EVALIDATION:
        raise (PlanError if plan else ValidationError)(msg)
    if rc == _abi.FPB_EFORMAT:
        raise FormatError(msg)
    if rc == _abi.FPB_ECUDA:
        raise CudaError(msg)
    raise ValueError(msg)


# ----------------------------------------------------------------------------- core.hpp

kLog2e = 1.4426950408889634  # core.hpp:13
kDefaultEpsilon = 1e-10  # core.hpp:14
kNegSentinel = -3.4028234663852886e38  # discovery.hpp:12 (FLT_LOWEST)


@dataclass(frozen=True)
class BlockGrid:
    """core.hpp:17-29."""

    block_size: int
    num_query_blocks: int
    num_key_blocks: int
    last_block_len: int

    def block_len(self, block: int) -> int:
        return self.last_block_len if block + 1 == self.num_key_blocks else self.block_size

    def block_of(self, token: int) -> int:
        return token // self.block_size


def make_block_grid(seq_len: int, block_size: int) -> BlockGrid:
    """core.hpp:31-41."""
    if seq_len < 1:
        raise ValidationError("sequence length must be >= 1")
    if block_size < 1:
        raise ValidationError("block size must be >= 1")
    blocks = (seq_len + block_size - 1) // block_size
    return BlockGrid(block_size, blocks, blocks, seq_len - (blocks - 1) * block_size)


@dataclass
class PipelineConfig:
    """core.hpp:87-112."""

    block_size: int = 128
    alpha: float = 0.12
    sink_tokens: int = 256
    window_tokens: int = 512
    scale: float = 0.0
    epsilon: float = kDefaultEpsilon
    rng_seed: int = 0

    def validate(self) -> None:
        if self.block_size < 1:
            raise ConfigError("block_size must be >= 1")
        if not (self.alpha >= 0.0):
            raise ConfigError("alpha must be >= 0")
        if self.window_tokens < 1:
            raise ConfigError("window_tokens must be >= 1")
        if not (self.epsilon > 0.0):
            raise ConfigError("epsilon must be > 0")

    def sink_blocks(self) -> int:
        return (self.sink_tokens + self.block_size - 1) // self.block_size

    def window_blocks(self) -> int:
        return (self.window_tokens + self.block_size - 1) // self.block_size

    def resolved_scale(self, head_dim: int) -> float:
        if self.scale > 0:
            return self.scale
        return float(torch.tensor(1.0, dtype=torch.float32) /
                     torch.sqrt(torch.tensor(float(head_dim), dtype=torch.float32)))


# ----------------------------------------------------------------------------- result types
# discovery.hpp:16-34, selection.hpp:14-38, attention.hpp:14-21


@dataclass
class PooledKeys:
    data: torch.Tensor  # Z x Hkv x N x d fp32


@dataclass
class BlockEnergies:
    energy: torch.Tensor
    local_max: torch.Tensor


@dataclass
class BlockScoreMap:
    energy: torch.Tensor | None
    local_max: torch.Tensor | None
    score: torch.Tensor


@dataclass
class ActiveMask:
    active: torch.Tensor  # Z x M x N x H u8


@dataclass
class SparseBlockPlan:
    indices: torch.Tensor  # Z x M x N x H i32
    counts: torch.Tensor  # Z x M x H i32


@dataclass
class SelectionStats:
    score_comparisons: int = 0


@dataclass
class AttentionOutput:
    out: torch.Tensor
    lse: torch.Tensor


@dataclass
class AttentionStats:
    block_visits: int = 0


# ----------------------------------------------------------------------------- plumbing


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _abi.FPB_BF16
    if t.dtype == torch.float32:
        return _abi.FPB_F32
    raise ValidationError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _dev(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValidationError(f"{name} must be contiguous")
    return t


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def problem(q_shape, hkv: int, config: PipelineConfig | None = None, tau: float | None = None,
            eps: float | None = None) -> _abi.Problem:
    Z, Hq, L, d = (int(x) for x in q_shape)
    p = _abi.Problem()
    _abi.lib().fpb_problem_init(C.byref(p), Z, Hq, hkv, L, d)
    if config is not None:
        p.block_size, p.alpha = config.block_size, config.alpha
        p.sink_tokens, p.window_tokens = config.sink_tokens, config.window_tokens
        p.scale, p.epsilon = config.scale, config.epsilon
    if tau is not None:
        p.scale = tau
    if eps is not None:
        p.epsilon = eps
    return p


_ws_cache: dict = {}
_ws_lock = threading.Lock()


def workspace(p: _abi.Problem, dtype_code: int, device) -> tuple[torch.Tensor | None, int]:
    """Grow-only scratch (fpb_workspace_bytes) per (device, current stream); no allocation on
    repeat calls.  The kernels keep their work-queue counters and list scratch in it, so calls on
    different streams must not share one buffer (reentrancy across streams); calls on
    one stream are ordered by the stream.  The buffer is allocated while its stream is current,
    so the caching allocator's reuse after a grow is ordered on that same stream."""
    n = C.c_size_t(0)
    _raise(_abi.lib().fpb_workspace_bytes(C.byref(p), dtype_code, C.byref(n)), "workspace")
    if n.value == 0:
        return None, 0
    dev = torch.device(device)
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    with _ws_lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < n.value:
            buf = torch.empty(n.value, dtype=torch.uint8, device=dev)
            _ws_cache[key] = buf
    return buf, n.value


def _check_qk(q: torch.Tensor, k: torch.Tensor):
    _dev(q, "queries")
    _dev(k, "keys")
    if q.dim() != 4 or k.dim() != 4:
        raise ValidationError("sequence batch must be Z x H x L x d")
    if q.dtype != k.dtype:
        raise ValidationError("query/key dtype mismatch")
    Z, Hq, L, d = q.shape
    if k.shape[0] != Z or k.shape[2] != L or k.shape[3] != d or Hq % k.shape[1]:
        raise ValidationError("query/key shape mismatch")  # core.hpp:81-85 (+ GQA)


def make_sequence_batch(data: torch.Tensor) -> torch.Tensor:
    """core.hpp:71-79: rejects non-4D shapes and non-finite values."""
    if data.dim() != 4 or min(data.shape) < 1:
        raise ValidationError("sequence batch must be Z x H x L x d")
    if not bool(torch.isfinite(data).all()):
        raise ValidationError("non-finite value in sequence batch")
    return data


# ----------------------------------------------------------------------------- discovery.hpp


def pool_keys(keys: torch.Tensor, grid: BlockGrid) -> PooledKeys:
    """discovery.hpp:65-70."""
    _dev(keys, "keys")
    Z, H, L, d = keys.shape
    if grid.num_key_blocks * grid.block_size < L:
        raise ValidationError("grid does not cover the key sequence")
    p = problem((Z, H, L, d), H)
    p.block_size = grid.block_size
    out = torch.empty((Z, H, grid.num_key_blocks, d), dtype=torch.float32, device=keys.device)
    _raise(_abi.lib().fpb_pool_keys(C.byref(p), _dtype_code(keys), _ptr(keys), _ptr(out),
                                    _stream(keys)), "pool_keys")
    return PooledKeys(out)


def approx_block_scores(queries: torch.Tensor, pooled: PooledKeys, grid: BlockGrid,
                        tau: float) -> BlockEnergies:
    """discovery.hpp:75-115."""
    _dev(queries, "queries")
    Z, Hq, L, d = queries.shape
    pk = _dev(pooled.data, "pooled")
    M = grid.num_query_blocks
    if pk.dim() != 4 or pk.shape[0] != Z or pk.shape[2] != M or pk.shape[3] != d or Hq % pk.shape[1]:
        raise ValidationError("pooled keys shape mismatch")
    p = problem(queries.shape, pk.shape[1], tau=tau)
    p.block_size = grid.block_size
    en = torch.empty((Z, Hq, M, M), dtype=torch.float32, device=queries.device)
    lm = torch.empty_like(en)
    ws, nws = workspace(p, _dtype_code(queries), queries.device)
    _raise(_abi.lib().fpb_approx_block_scores(C.byref(p), _dtype_code(queries), _ptr(queries),
                                              _ptr(pk), _ptr(en), _ptr(lm), _ptr(ws), nws,
                                              _stream(queries)), "approx_block_scores")
    return BlockEnergies(en, lm)


def normalize_block_scores(energies: BlockEnergies, grid: BlockGrid,
                           epsilon: float = kDefaultEpsilon) -> BlockScoreMap:
    """discovery.hpp:119-148."""
    en, lm = _dev(energies.energy, "energy"), _dev(energies.local_max, "local_max")
    Z, H, M, _ = en.shape
    p = problem((Z, H, (M - 1) * grid.block_size + grid.last_block_len, 128), H, eps=epsilon)
    p.block_size = grid.block_size
    score = torch.empty_like(en)
    _raise(_abi.lib().fpb_normalize_block_scores(C.byref(p), _ptr(en), _ptr(lm), _ptr(score),
                                                 _stream(en)), "normalize_block_scores")
    return BlockScoreMap(en, lm, score)


def discover(queries: torch.Tensor, keys: torch.Tensor, grid: BlockGrid, tau: float,
             epsilon: float = kDefaultEpsilon, maps: bool = True) -> BlockScoreMap:
    """discovery.hpp:153-159 (pooling + approximation + normalisation: one discovery launch for
    bf16 keys, which pools K in-kernel; fp32 keys are pooled by a separate launch).

    maps=False skips materialising energy/local_max (score only)."""
    _check_qk(queries, keys)
    Z, Hq, L, d = queries.shape
    M = grid.num_query_blocks
    p = problem(queries.shape, keys.shape[1], tau=tau, eps=epsilon)
    p.block_size = grid.block_size
    dev = queries.device
    score = torch.empty((Z, Hq, M, M), dtype=torch.float32, device=dev)
    en = torch.empty_like(score) if maps else None
    lm = torch.empty_like(score) if maps else None
    ws, nws = workspace(p, _dtype_code(queries), dev)
    _raise(_abi.lib().fpb_discover(C.byref(p), _dtype_code(queries), _ptr(queries), _ptr(keys),
                                   _ptr(en), _ptr(lm), _ptr(score), _ptr(ws), nws,
                                   _stream(queries)), "discover")
    return BlockScoreMap(en, lm, score)


# ----------------------------------------------------------------------------- selection.hpp


def max_threshold_mask(scores, config: PipelineConfig,
                       stats: SelectionStats | None = None) -> ActiveMask:
    """selection.hpp:63-92 (and the BlockScoreMap overload, :161-164)."""
    config.validate()
    score = scores.score if isinstance(scores, BlockScoreMap) else scores
    _dev(score, "score")
    if score.dim() != 4:
        raise ValidationError("score map must be Z x H x M x N")
    Z, H, M, N = score.shape
    if M != N:
        raise ValidationError("score map must be square (M == N)")
    p = problem((Z, H, (M - 1) * config.block_size + 1, 128), H, config=config)
    mask = torch.empty((Z, M, N, H), dtype=torch.uint8, device=score.device)
    cmp = torch.zeros(1, dtype=torch.int64, device=score.device) if stats is not None else None
    _raise(_abi.lib().fpb_max_threshold_mask(C.byref(p), _ptr(score), _ptr(mask), _ptr(cmp),
                                             _stream(score)), "max_threshold_mask")
    if stats is not None:
        stats.score_comparisons += int(cmp.item())
    return ActiveMask(mask)


def compress_indices(mask: ActiveMask) -> SparseBlockPlan:
    """selection.hpp:176-192."""
    m = _dev(mask.active, "mask")
    Z, M, N, H = m.shape
    p = problem((Z, H, (M - 1) * 128 + 1, 128), H)
    idx = torch.empty((Z, M, N, H), dtype=torch.int32, device=m.device)
    counts = torch.empty((Z, M, H), dtype=torch.int32, device=m.device)
    _raise(_abi.lib().fpb_compress_indices(C.byref(p), _ptr(m), _ptr(idx), _ptr(counts),
                                           _stream(m)), "compress_indices")
    return SparseBlockPlan(idx, counts)


def _sort_select(scores, config: PipelineConfig, mode: int, k: int = 1, p: float = 1.0):
    config.validate()
    score = scores.score if isinstance(scores, BlockScoreMap) else scores
    _dev(score, "score")
    Z, H, M, N = score.shape
    pr = problem((Z, H, (M - 1) * config.block_size + 1, 128), H, config=config)
    mask = torch.empty((Z, M, N, H), dtype=torch.uint8, device=score.device)
    fn = _abi.lib().fpb_topk_select if mode == 0 else _abi.lib().fpb_topp_select
    arg = C.c_int32(k) if mode == 0 else C.c_float(p)
    rc = fn(C.byref(pr), _ptr(score), arg, _ptr(mask), _stream(score))
    if rc == _abi.FPB_EVALIDATION:
        raise ConfigError(_abi.last_error())
    _raise(rc, "topk_select" if mode == 0 else "topp_select")
    return ActiveMask(mask)


def topk_select(scores, k: int, config: PipelineConfig) -> ActiveMask:
    """selection.hpp:96-123 (comparison baseline): min(k, i+1) top blocks per causal row, ties
    toward the lower index, plus sink/window retention."""
    if k < 1:
        raise ConfigError("top-k requires k >= 1")
    return _sort_select(scores, config, 0, k=k)


def topp_select(scores, p: float, config: PipelineConfig) -> ActiveMask:
    """selection.hpp:127-159 (comparison baseline): shortest descending prefix reaching mass p."""
    if not (p > 0.0) or p > 1.0:
        raise ConfigError("top-p requires p in (0, 1]")
    return _sort_select(scores, config, 1, p=p)


def _baseline_discover(fn, name, queries, keys, grid, tau, epsilon):
    _check_qk(queries, keys)
    Z, Hq, L, d = queries.shape
    M = grid.num_query_blocks
    pr = problem(queries.shape, keys.shape[1], tau=tau, eps=epsilon)
    pr.block_size = grid.block_size
    n = C.c_size_t(0)
    _raise(_abi.lib().fpb_baseline_workspace_bytes(C.byref(pr), C.byref(n)), name)
    ws = torch.empty(max(1, n.value), dtype=torch.uint8, device=queries.device)
    en = torch.empty((Z, Hq, M, M), dtype=torch.float32, device=queries.device)
    lm, sc = torch.empty_like(en), torch.empty_like(en)
    _raise(fn(C.byref(pr), _dtype_code(queries), _ptr(queries), _ptr(keys), _ptr(en), _ptr(lm),
              _ptr(sc), _ptr(ws), n.value, _stream(queries)), name)
    return BlockScoreMap(en, lm, sc)


def discover_pool_both(queries, keys, grid: BlockGrid, tau: float,
                       epsilon: float = kDefaultEpsilon) -> BlockScoreMap:
    """discovery.hpp:164-195 (comparison method): mean-pool Q as well."""
    return _baseline_discover(_abi.lib().fpb_discover_pool_both, "discover_pool_both", queries,
                              keys, grid, tau, epsilon)


def discover_exact(queries, keys, grid: BlockGrid, tau: float,
                   epsilon: float = kDefaultEpsilon) -> BlockScoreMap:
    """discovery.hpp:201-279 (reference semantics): per-query softmax over pooled keys, averaged
    over each query block."""
    return _baseline_discover(_abi.lib().fpb_discover_exact, "discover_exact", queries, keys,
                              grid, tau, epsilon)


def visit_count(plan: SparseBlockPlan) -> int:
    """selection.hpp:195-200."""
    c = _dev(plan.counts, "counts")
    Z, M, H = c.shape
    p = problem((Z, H, (M - 1) * 128 + 1, 128), H)
    total = torch.zeros(1, dtype=torch.int64, device=c.device)
    _raise(_abi.lib().fpb_visit_count(C.byref(p), _ptr(c), _ptr(total), _stream(c)), "visit_count")
    return int(total.item())


def density(plan: SparseBlockPlan, grid: BlockGrid) -> float:
    """selection.hpp:203-209."""
    Z, _, H = plan.counts.shape
    M = grid.num_query_blocks
    return visit_count(plan) / (Z * H * (M * (M + 1) / 2.0))


def _rows_args(rows):
    """(entry-point suffix, a, b) of a row shard: (row_begin, row_step) for the interleaved shard
    (fpb_*_rows), ("zigzag", rank, world) for the zigzag shard (fpb_*_zigzag)."""
    if len(rows) == 3 and rows[0] == "zigzag":
        return "zigzag", int(rows[1]), int(rows[2])
    return "rows", int(rows[0]), int(rows[1])


def discover_select(queries: torch.Tensor, keys: torch.Tensor, config: PipelineConfig,
                    want_score: bool = False, want_mask: bool = False,
                    want_energy: bool = False, rows: tuple[int, int] | None = None):
    """Fused discover -> max_threshold_mask -> compress_indices (one pass over Q).

    rows=(row_begin, row_step) restricts the work to query blocks row_begin + row_step * k
    (fpb_discover_select_rows, the row-sharded multi-GPU partition); rows=("zigzag", rank, world)
    to rank's two contiguous chunks (fpb_discover_select_zigzag); rows of other blocks in the
    returned tensors are left unwritten.
    Returns (SparseBlockPlan, BlockScoreMap | None, ActiveMask | None)."""
    config.validate()
    _check_qk(queries, keys)
    Z, Hq, L, d = queries.shape
    grid = make_block_grid(L, config.block_size)
    M = grid.num_query_blocks
    dev = queries.device
    p = problem(queries.shape, keys.shape[1], config=config)
    idx = torch.empty((Z, M, M, Hq), dtype=torch.int32, device=dev)
    counts = torch.empty((Z, M, Hq), dtype=torch.int32, device=dev)
    score = torch.empty((Z, Hq, M, M), dtype=torch.float32, device=dev) if want_score else None
    en = torch.empty((Z, Hq, M, M), dtype=torch.float32, device=dev) if want_energy else None
    lm = torch.empty_like(en) if want_energy else None
    mask = torch.empty((Z, M, M, Hq), dtype=torch.uint8, device=dev) if want_mask else None
    ws, nws = workspace(p, _dtype_code(queries), dev)
    if rows is None:
        _raise(_abi.lib().fpb_discover_select(C.byref(p), _dtype_code(queries), _ptr(queries),
                                              _ptr(keys), _ptr(en), _ptr(lm), _ptr(score),
                                              _ptr(mask), _ptr(idx), _ptr(counts), _ptr(ws), nws,
                                              _stream(queries)), "discover_select")
    else:
        kind, a, b = _rows_args(rows)
        _raise(getattr(_abi.lib(), f"fpb_discover_select_{kind}")(
            C.byref(p), a, b, _dtype_code(queries), _ptr(queries),
            _ptr(keys), _ptr(en), _ptr(lm), _ptr(score), _ptr(mask), _ptr(idx), _ptr(counts),
            _ptr(ws), nws, _stream(queries)), f"discover_select_{kind}")
    smap = BlockScoreMap(en, lm, score) if want_score else None
    return SparseBlockPlan(idx, counts), smap, (ActiveMask(mask) if want_mask else None)


# ----------------------------------------------------------------------------- attention.hpp


def _check_qkv(q, k, v):
    _check_qk(q, k)
    _dev(v, "values")
    if v.shape != k.shape or v.dtype != k.dtype:
        raise ValidationError("key/value shape mismatch")


def _out_code(out_dtype, q):
    out_dtype = out_dtype or q.dtype
    return out_dtype, (_abi.FPB_BF16 if out_dtype == torch.bfloat16 else _abi.FPB_F32)


def block_sparse_attention(queries, keys, values, plan: SparseBlockPlan, grid: BlockGrid,
                           tau: float, stats: AttentionStats | None = None,
                           out_dtype: torch.dtype | None = None,
                           rows: tuple[int, int] | None = None) -> AttentionOutput:
    """attention.hpp:38-132.  Raises PlanError for a block index outside [0, N).

    rows=(row_begin, row_step): only query blocks row_begin + row_step * k are computed
    (fpb_block_sparse_attention_rows); rows=("zigzag", rank, world): rank's zigzag chunks
    (fpb_block_sparse_attention_zigzag); output rows of other blocks are left unwritten."""
    _check_qkv(queries, keys, values)
    Z, Hq, L, d = queries.shape
    M = grid.num_query_blocks
    idx, counts = _dev(plan.indices, "indices"), _dev(plan.counts, "counts")
    if tuple(idx.shape) != (Z, M, M, Hq) or tuple(counts.shape) != (Z, M, Hq):
        raise ValidationError("plan shape does not match grid/batch")
    p = problem(queries.shape, keys.shape[1], tau=tau)
    p.block_size = grid.block_size
    dev = queries.device
    out_dtype, oc = _out_code(out_dtype, queries)
    out = torch.empty(queries.shape, dtype=out_dtype, device=dev)
    lse = torch.empty((Z, Hq, L), dtype=torch.float32, device=dev)
    aux = torch.zeros(2, dtype=torch.int64, device=dev)  # [visits, plan_error]
    ws, nws = workspace(p, _dtype_code(queries), dev)
    if rows is None:
        _raise(_abi.lib().fpb_block_sparse_attention(
            C.byref(p), _dtype_code(queries), _ptr(queries), _ptr(keys), _ptr(values), _ptr(idx),
            _ptr(counts), oc, _ptr(out), _ptr(lse), C.c_void_p(aux.data_ptr()),
            C.c_void_p(aux.data_ptr() + 8), _ptr(ws), nws, _stream(queries)),
            "block_sparse_attention")
    else:
        kind, a, b = _rows_args(rows)
        _raise(getattr(_abi.lib(), f"fpb_block_sparse_attention_{kind}")(
            C.byref(p), a, b, _dtype_code(queries), _ptr(queries),
            _ptr(keys), _ptr(values), _ptr(idx), _ptr(counts), oc, _ptr(out), _ptr(lse),
            C.c_void_p(aux.data_ptr()), C.c_void_p(aux.data_ptr() + 8), _ptr(ws), nws,
            _stream(queries)), f"block_sparse_attention_{kind}")
    visits, err = (int(x) for x in aux.tolist())
    if err:
        raise PlanError(f"plan row lists a block index outside [0, {M})")
    if stats is not None:
        stats.block_visits += visits
    return AttentionOutput(out, lse)


def dense_attention(queries, keys, values, tau: float,
                    out_dtype: torch.dtype | None = None) -> AttentionOutput:
    """attention.hpp:135-174 — the dense causal kernel (speedup denominator)."""
    _check_qkv(queries, keys, values)
    Z, Hq, L, d = queries.shape
    p = problem(queries.shape, keys.shape[1], tau=tau)
    dev = queries.device
    out_dtype, oc = _out_code(out_dtype, queries)
    out = torch.empty(queries.shape, dtype=out_dtype, device=dev)
    lse = torch.empty((Z, Hq, L), dtype=torch.float32, device=dev)
    ws, nws = workspace(p, _dtype_code(queries), dev)
    _raise(_abi.lib().fpb_dense_attention(C.byref(p), _dtype_code(queries), _ptr(queries),
                                          _ptr(keys), _ptr(values), oc, _ptr(out), _ptr(lse),
                                          _ptr(ws), nws, _stream(queries)), "dense_attention")
    return AttentionOutput(out, lse)


def full_causal_plan(batch: int, heads: int, grid: BlockGrid, device="cuda") -> SparseBlockPlan:
    """attention.hpp:178-192."""
    M = grid.num_query_blocks
    p = problem((batch, heads, (M - 1) * grid.block_size + 1, 128), heads)
    p.block_size = grid.block_size
    idx = torch.empty((batch, M, M, heads), dtype=torch.int32, device=device)
    counts = torch.empty((batch, M, heads), dtype=torch.int32, device=device)
    _raise(_abi.lib().fpb_full_causal_plan(C.byref(p), _ptr(idx), _ptr(counts),
                                           C.c_void_p(torch.cuda.current_stream(device).cuda_stream)),
           "full_causal_plan")
    return SparseBlockPlan(idx, counts)


def prefill(queries, keys, values, config: PipelineConfig,
            out_dtype: torch.dtype | None = None, stats: AttentionStats | None = None):
    """The whole FlashPrefill step (acceptance.cpp:357-360) on device tensors:
    fused discover+select, then block-sparse attention.  Returns (AttentionOutput, plan)."""
    plan, _, _ = discover_select(queries, keys, config)
    grid = make_block_grid(queries.shape[2], config.block_size)
    tau = config.resolved_scale(queries.shape[3])
    return block_sparse_attention(queries, keys, values, plan, grid, tau, stats, out_dtype), plan


def prefill_host(q_host, k_host, v_host, config: PipelineConfig, out_host, lse_host,
                 idx_host=None, counts_host=None) -> int:
    """fpb_host_prefill over HOST tensors (pinned recommended): H2D, kernels, D2H, sync.

    Returns block visits.  This is the reference-facing end-to-end call bench.py times."""
    for t in (q_host, k_host, v_host, out_host, lse_host):
        if t.is_cuda or not t.is_contiguous():
            raise ValidationError("prefill_host takes contiguous host tensors")
    p = problem(q_host.shape, k_host.shape[1], config=config)
    vis = C.c_uint64(0)
    oc = _abi.FPB_BF16 if out_host.dtype == torch.bfloat16 else _abi.FPB_F32
    _raise(_abi.lib().fpb_host_prefill(C.byref(p), _dtype_code(q_host), _ptr(q_host),
                                       _ptr(k_host), _ptr(v_host), oc, _ptr(out_host),
                                       _ptr(lse_host), _ptr(idx_host), _ptr(counts_host),
                                       C.byref(vis)), "prefill_host")
    return vis.value


def flops_dense_causal(Z: int, Hq: int, L: int, d: int) -> float:
    """Dense-causal-equivalent attention FLOPs: 4 d Z Hq L(L+1)/2."""
    return 4.0 * d * Z * Hq * L * (L + 1) / 2.0


def flops_sparse(visits_off_diag: int, visits_diag: int, d: int = 128, B: int = 128) -> float:
    """Algorithmic FLOPs of the visited blocks: 4 d B^2 per off-diagonal visit, 4 d B(B+1)/2 per
    diagonal visit."""
    return 4.0 * d * (visits_off_diag * B * B + visits_diag * B * (B + 1) / 2.0)



# ----------------------------------------------------------------------------- device-resident step
class PrefillRunner:
    """The device-resident FlashPrefill step with preallocated buffers, for serving loops and the
    benchmark: fpb_discover_select then fpb_block_sparse_attention on the current stream, no host
    allocation and no host synchronisation per step (the Python wrappers above sync once per call
    to raise PlanError like the reference).  capture() records each stage into a CUDA graph, so a
    step is two graph launches (the launch-bound inner loop without a tracing compiler).

    rows=(row_begin, row_step) runs one rank's row shard (fpb_*_rows), rows=("zigzag", rank, world)
    its zigzag shard (fpb_*_zigzag)."""

    def __init__(self, queries, keys, values, config: PipelineConfig,
                 out_dtype: torch.dtype = torch.bfloat16, rows: tuple[int, int] | None = None):
        config.validate()
        _check_qkv(queries, keys, values)
        self.q, self.k, self.v = queries, keys, values
        Z, Hq, L, d = queries.shape
        self.grid = make_block_grid(L, config.block_size)
        M = self.grid.num_query_blocks
        dev = queries.device
        self.p = problem(queries.shape, keys.shape[1], config=config)
        self.dt = _dtype_code(queries)
        self.out_dtype, self.oc = _out_code(out_dtype, queries)
        self.rows = rows
        self.idx = torch.empty((Z, M, M, Hq), dtype=torch.int32, device=dev)
        self.counts = torch.empty((Z, M, Hq), dtype=torch.int32, device=dev)
        self.out = torch.empty(queries.shape, dtype=self.out_dtype, device=dev)
        self.lse = torch.empty((Z, Hq, L), dtype=torch.float32, device=dev)
        self.aux = torch.zeros(2, dtype=torch.int64, device=dev)  # [visits, plan_error]
        n = C.c_size_t(0)
        _raise(_abi.lib().fpb_workspace_bytes(C.byref(self.p), self.dt, C.byref(n)), "workspace")
        self.nws = n.value
        self.ws = torch.empty(max(1, n.value), dtype=torch.uint8, device=dev)
        self.graphs = None

    @property
    def plan(self) -> SparseBlockPlan:
        return SparseBlockPlan(self.idx, self.counts)

    def discover(self):
        lib, s = _abi.lib(), _stream(self.q)
        if self.rows is None:
            rc = lib.fpb_discover_select(C.byref(self.p), self.dt, _ptr(self.q), _ptr(self.k),
                                         None, None, None, None, _ptr(self.idx),
                                         _ptr(self.counts), _ptr(self.ws), self.nws, s)
        else:
            kind, a, b = _rows_args(self.rows)
            rc = getattr(lib, f"fpb_discover_select_{kind}")(
                C.byref(self.p), a, b, self.dt, _ptr(self.q), _ptr(self.k), None, None, None, None,
                _ptr(self.idx), _ptr(self.counts), _ptr(self.ws), self.nws, s)
        _raise(rc, "discover_select")

    def attend(self):
        lib, s = _abi.lib(), _stream(self.q)
        vis, err = C.c_void_p(self.aux.data_ptr()), C.c_void_p(self.aux.data_ptr() + 8)
        if self.rows is None:
            rc = lib.fpb_block_sparse_attention(
                C.byref(self.p), self.dt, _ptr(self.q), _ptr(self.k), _ptr(self.v), _ptr(self.idx),
                _ptr(self.counts), self.oc, _ptr(self.out), _ptr(self.lse), vis, err,
                _ptr(self.ws), self.nws, s)
        else:
            kind, a, b = _rows_args(self.rows)
            rc = getattr(lib, f"fpb_block_sparse_attention_{kind}")(
                C.byref(self.p), a, b, self.dt, _ptr(self.q), _ptr(self.k),
                _ptr(self.v), _ptr(self.idx), _ptr(self.counts), self.oc, _ptr(self.out),
                _ptr(self.lse), vis, err, _ptr(self.ws), self.nws, s)
        _raise(rc, "block_sparse_attention")

    def capture(self):
        """Record discover and attend into two CUDA graphs (warm-up launch first)."""
        side = torch.cuda.Stream(self.q.device)
        side.wait_stream(torch.cuda.current_stream(self.q.device))
        with torch.cuda.stream(side):
            self.discover()
            self.attend()
        torch.cuda.current_stream(self.q.device).wait_stream(side)
        torch.cuda.synchronize(self.q.device)
        # keep_graph: the cudaGraph_t stays queryable (kernel_nodes) after instantiation
        g_disc, g_attn = torch.cuda.CUDAGraph(keep_graph=True), torch.cuda.CUDAGraph(keep_graph=True)
        # relaxed: the launch helpers query device attributes while the stream is capturing
        with torch.cuda.graph(g_disc, capture_error_mode="relaxed"):
            self.discover()
        with torch.cuda.graph(g_attn, capture_error_mode="relaxed"):
            self.attend()
        g_disc.instantiate()
        g_attn.instantiate()
        self.graphs = (g_disc, g_attn)
        return self

    def replay_discover(self):
        if self.graphs:
            self.graphs[0].replay()
        else:
            self.discover()

    def replay_attend(self):
        if self.graphs:
            self.graphs[1].replay()
        else:
            self.attend()

    def check(self) -> int:
        """Synchronises; raises PlanError if any replay saw an out-of-range block index and
        returns the accumulated block visits."""
        visits, err = (int(x) for x in self.aux.tolist())
        if err:
            raise PlanError(f"plan row lists a block index outside [0, {self.grid.num_query_blocks})")
        return visits
