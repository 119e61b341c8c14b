"""CPU parity oracle for the FlashPrefill hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the cpu_baseline / reference leg of ``bench.py``
may import this package.  It wraps two shared libraries with numpy-facing functions of identical
signatures:

* ``liboracle.so`` (``oracle/bsattn_oracle.c``): the C restatement of the reference algorithm, each
  function citing the reference file:line it follows.
* ``_ref/libbsattn_ref.so`` (``oracle/ref_shim.cpp``): the UNMODIFIED reference headers
  (/root/reference/proj/include/bsattn) behind an ``extern "C"`` shim.

``Oracle("port")`` / ``Oracle("reference")`` select the implementation; both expose the same
methods so tests can pin one against the other.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libbsattn_ref.so")

_u64, _u32, _i64, _f32, _i32 = C.c_uint64, C.c_uint32, C.c_int64, C.c_float, C.c_int
_p = C.c_void_p

LOG2E = np.float32(1.4426950408889634)
NEG_SENTINEL = np.finfo(np.float32).min


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and _ref when /root/reference exists) with oracle/Makefile."""
    out = subprocess.run(["make", "-C", _HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


def _ptr(a):
    return a.ctypes.data_as(_p) if a is not None else None


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Oracle:
    """numpy front-end over liboracle.so ("port") or the reference shim ("reference")."""

    def __init__(self, kind: str = "port"):
        if kind not in ("port", "reference"):
            raise ValueError(kind)
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            if kind == "port":
                build()
            else:
                raise FileNotFoundError(f"{path} missing (reference headers absent at build time)")
        self.lib = C.CDLL(path)
        pre = "or_" if kind == "port" else "ref_"
        self._fn = lambda name: getattr(self.lib, pre + name)
        self._setup(pre)

    def _setup(self, pre):
        L = self.lib
        gp = lambda n: getattr(L, pre + n)
        gp("pool_keys").argtypes = [_p, _u64, _u64, _u64, _u64, _u32, _p]
        gp("max_threshold_mask").argtypes = [_p, _u64, _u64, _u32, _u32, _u32, _f32, _u32, _u32,
                                             _f32, _p, _p]
        gp("compress_indices").argtypes = [_p, _u64, _u32, _u32, _u64, _p, _p]
        gp("generate_planted").argtypes = [_i32, _f32, _i64, _i64, _f32, _u64, _u64, _u64, _u64,
                                           _u64, _u32, _f32, _p, _p, _p, _p]
        gp("pipeline_threads").argtypes = [_p, _p, _p, _u64, _u64, _u64, _u64, _u64, _u32, _f32,
                                           _u32, _u32, _f32, _f32, _p, _i32, _i32, _p, _p, _p]
        gp("pipeline_threads").restype = C.c_double
        if pre == "ref_":
            gp("pipeline_detail").argtypes = [_p, _p, _p, _u64, _u64, _u64, _u64, _u64, _u32,
                                              _f32, _u32, _u32, _f32, _f32, _p, _i32, _i32, _p,
                                              _p, _p, _p, _p, _p, _p, _p]
            gp("pipeline_detail").restype = C.c_double
        gp("topk_select").argtypes = [_p, _u64, _u64, _u32, _u32, _u32, _u32, _u32, _p]
        gp("topp_select").argtypes = [_p, _u64, _u64, _u32, _f32, _u32, _u32, _u32, _p]
        if pre == "or_":
            gp("discover_pool_both").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u64, _u32, _f32,
                                                 _f32, _p, _p, _p]
            gp("discover_exact").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u64, _u32, _f32,
                                             _f32, _p, _p, _p]
        else:
            gp("discover_pool_both").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u32, _f32, _f32,
                                                 _p, _p, _p]
            gp("discover_exact").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u32, _f32, _f32, _p,
                                             _p, _p]
        if pre == "or_":
            gp("discover").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u64, _u32, _f32, _f32, _p,
                                       _p, _p]
            gp("approx_block_scores").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u64, _u32, _f32,
                                                  _p, _p]
            gp("normalize_block_scores").argtypes = [_p, _p, _u64, _u64, _u32, _f32, _p]
            gp("block_sparse_attention").argtypes = [_p, _p, _p, _u64, _u64, _u64, _u64, _u64,
                                                     _u32, _p, _p, _f32, _p, _p, _p]
            gp("dense_attention").argtypes = [_p, _p, _p, _u64, _u64, _u64, _u64, _u64, _f32, _p,
                                              _p]
            gp("full_causal_plan").argtypes = [_u64, _u64, _u32, _p, _p]
            gp("random_batch").argtypes = [_u64, _u64, _f32, _p]
        else:
            gp("discover").argtypes = [_p, _p, _u64, _u64, _u64, _u64, _u32, _f32, _f32, _p, _p,
                                       _p]
            gp("block_sparse_attention").argtypes = [_p, _p, _p, _u64, _u64, _u64, _u64, _u32, _p,
                                                     _p, _f32, _p, _p, _p]
            gp("dense_attention").argtypes = [_p, _p, _p, _u64, _u64, _u64, _u64, _f32, _p, _p]

    # ------------------------------------------------------------------ helpers
    @staticmethod
    def grid(L: int, B: int):
        M = (L + B - 1) // B
        return M, L - (M - 1) * B

    @staticmethod
    def scale(d: int, scale: float = 0.0) -> np.float32:
        return np.float32(scale) if scale > 0 else np.float32(1.0) / np.sqrt(np.float32(d))

    @staticmethod
    def _check(rc, what):
        if rc != 0:
            raise ValueError(f"{what} failed with code {rc}")

    # ------------------------------------------------------------------ hot path
    def pool_keys(self, k, B):
        k = _f(k)
        Z, H, L, d = k.shape
        M, _ = self.grid(L, B)
        out = np.empty((Z, H, M, d), np.float32)
        self._check(self._fn("pool_keys")(_ptr(k), Z, H, L, d, B, _ptr(out)), "pool_keys")
        return out

    def discover(self, q, k, B, tau, eps=1e-10):
        """Returns (energy, local_max, score), each Z x Hq x M x N."""
        q, k = _f(q), _f(k)
        Z, Hq, L, d = q.shape
        Hkv = k.shape[1]
        M, _ = self.grid(L, B)
        en = np.empty((Z, Hq, M, M), np.float32)
        lm = np.empty_like(en)
        sc = np.empty_like(en)
        if self.kind == "port":
            rc = self._fn("discover")(_ptr(q), _ptr(k), Z, Hq, Hkv, L, d, B, tau, eps, _ptr(en),
                                      _ptr(lm), _ptr(sc))
            self._check(rc, "discover")
        else:
            g = Hq // Hkv
            for z in range(Z):
                for h in range(Hq):
                    qs = np.ascontiguousarray(q[z, h])
                    ks = np.ascontiguousarray(k[z, h // g])
                    e1, l1, s1 = (np.empty((M, M), np.float32) for _ in range(3))
                    rc = self._fn("discover")(_ptr(qs), _ptr(ks), 1, 1, L, d, B, tau, eps,
                                              _ptr(e1), _ptr(l1), _ptr(s1))
                    self._check(rc, "discover")
                    en[z, h], lm[z, h], sc[z, h] = e1, l1, s1
        return en, lm, sc

    def sort_select(self, score, mode, param, B=128, sink_tokens=256, window_tokens=512):
        """topk_select (mode 'topk', param k) / topp_select (mode 'topp', param p)."""
        score = _f(score)
        Z, H, M, _ = score.shape
        mask = np.empty((Z, M, M, H), np.uint8)
        fn = self._fn("topk_select" if mode == "topk" else "topp_select")
        rc = fn(_ptr(score), Z, H, M, param, B, sink_tokens, window_tokens, _ptr(mask))
        self._check(rc, mode)
        return mask

    def discover_variant(self, method, q, k, B, tau, eps=1e-10):
        """discover_pool_both (method 'pool-both') / discover_exact (method 'exact')."""
        q, k = _f(q), _f(k)
        Z, Hq, L, d = q.shape
        Hkv = k.shape[1]
        M, _ = self.grid(L, B)
        en = np.empty((Z, Hq, M, M), np.float32)
        lm, sc = np.empty_like(en), np.empty_like(en)
        name = "discover_pool_both" if method == "pool-both" else "discover_exact"
        if self.kind == "port":
            rc = self._fn(name)(_ptr(q), _ptr(k), Z, Hq, Hkv, L, d, B, tau, eps, _ptr(en), _ptr(lm),
                                _ptr(sc))
            self._check(rc, name)
        else:
            g = Hq // Hkv
            for z in range(Z):
                for h in range(Hq):
                    qs = np.ascontiguousarray(q[z, h])
                    ks = np.ascontiguousarray(k[z, h // g])
                    e1, l1, s1 = (np.empty((M, M), np.float32) for _ in range(3))
                    rc = self._fn(name)(_ptr(qs), _ptr(ks), 1, 1, L, d, B, tau, eps, _ptr(e1),
                                        _ptr(l1), _ptr(s1))
                    self._check(rc, name)
                    en[z, h], lm[z, h], sc[z, h] = e1, l1, s1
        return en, lm, sc

    def max_threshold_mask(self, score, B=128, alpha=0.12, sink_tokens=256, window_tokens=512,
                           eps=1e-10):
        """Returns (mask Z x M x N x H u8, comparisons)."""
        score = _f(score)
        Z, H, M, N = score.shape
        mask = np.empty((Z, M, N, H), np.uint8)
        cmp = C.c_uint64(0)
        rc = self._fn("max_threshold_mask")(_ptr(score), Z, H, M, N, B, alpha, sink_tokens,
                                            window_tokens, eps, _ptr(mask), C.byref(cmp))
        self._check(rc, "max_threshold_mask")
        return mask, cmp.value

    def compress_indices(self, mask):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        Z, M, N, H = mask.shape
        idx = np.empty((Z, M, N, H), np.int32)
        counts = np.empty((Z, M, H), np.int32)
        self._check(self._fn("compress_indices")(_ptr(mask), Z, M, N, H, _ptr(idx), _ptr(counts)),
                    "compress_indices")
        return idx, counts

    def block_sparse_attention(self, q, k, v, idx, counts, B, tau):
        """Returns (out, lse, visits).  Raises ValueError on a PlanError."""
        q, k, v = _f(q), _f(k), _f(v)
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        Z, Hq, L, d = q.shape
        Hkv = k.shape[1]
        out = np.empty_like(q)
        lse = np.empty((Z, Hq, L), np.float32)
        vis = C.c_uint64(0)
        if self.kind == "port":
            rc = self._fn("block_sparse_attention")(_ptr(q), _ptr(k), _ptr(v), Z, Hq, Hkv, L, d, B,
                                                    _ptr(idx), _ptr(counts), tau, _ptr(out),
                                                    _ptr(lse), C.byref(vis))
            self._check(rc, "block_sparse_attention")
        else:
            g = Hq // Hkv
            for z in range(Z):
                for h in range(Hq):
                    qs = np.ascontiguousarray(q[z:z + 1, h:h + 1])
                    ks = np.ascontiguousarray(k[z:z + 1, h // g:h // g + 1])
                    vs = np.ascontiguousarray(v[z:z + 1, h // g:h // g + 1])
                    i1 = np.ascontiguousarray(idx[z:z + 1, :, :, h:h + 1])
                    c1 = np.ascontiguousarray(counts[z:z + 1, :, h:h + 1])
                    o1 = np.empty_like(qs)
                    l1 = np.empty((1, 1, L), np.float32)
                    rc = self._fn("block_sparse_attention")(_ptr(qs), _ptr(ks), _ptr(vs), 1, 1, L,
                                                            d, B, _ptr(i1), _ptr(c1), tau,
                                                            _ptr(o1), _ptr(l1), C.byref(vis))
                    self._check(rc, "block_sparse_attention")
                    out[z, h], lse[z, h] = o1[0, 0], l1[0, 0]
        return out, lse, vis.value

    def dense_attention(self, q, k, v, tau):
        q, k, v = _f(q), _f(k), _f(v)
        Z, Hq, L, d = q.shape
        Hkv = k.shape[1]
        out = np.empty_like(q)
        lse = np.empty((Z, Hq, L), np.float32)
        if self.kind == "port":
            self._check(self._fn("dense_attention")(_ptr(q), _ptr(k), _ptr(v), Z, Hq, Hkv, L, d,
                                                    tau, _ptr(out), _ptr(lse)), "dense_attention")
        else:
            g = Hq // Hkv
            for z in range(Z):
                for h in range(Hq):
                    qs = np.ascontiguousarray(q[z:z + 1, h:h + 1])
                    ks = np.ascontiguousarray(k[z:z + 1, h // g:h // g + 1])
                    vs = np.ascontiguousarray(v[z:z + 1, h // g:h // g + 1])
                    o1 = np.empty_like(qs)
                    l1 = np.empty((1, 1, L), np.float32)
                    self._check(self._fn("dense_attention")(_ptr(qs), _ptr(ks), _ptr(vs), 1, 1, L,
                                                            d, tau, _ptr(o1), _ptr(l1)),
                                "dense_attention")
                    out[z, h], lse[z, h] = o1[0, 0], l1[0, 0]
        return out, lse

    def generate_planted(self, kind, strength, a, b, noise, seed, Z, H, L, d, B, tau=0.0):
        """workloads.hpp generate_planted: returns (q, k, v, ground_truth Z x M x M x H)."""
        q = np.empty((Z, H, L, d), np.float32)
        k = np.empty_like(q)
        v = np.empty_like(q)
        M, _ = self.grid(L, B)
        gt = np.empty((Z, M, M, H), np.uint8)
        rc = self._fn("generate_planted")(kind, strength, a, b, noise, seed, Z, H, L, d, B, tau,
                                          _ptr(q), _ptr(k), _ptr(v), _ptr(gt))
        self._check(rc, "generate_planted")
        return q, k, v, gt

    def pipeline(self, q, k, v, B, alpha, sink_tokens, window_tokens, tau, eps, heads, threads):
        """Full pipeline per (z*Hq + h) slice in `heads` on `threads` threads.

        Returns (seconds, out[len(heads), L, d], lse[len(heads), L], visits)."""
        q, k, v = _f(q), _f(k), _f(v)
        Z, Hq, L, d = q.shape
        Hkv = k.shape[1]
        heads = np.ascontiguousarray(heads, dtype=np.int32)
        out = np.empty((len(heads), L, d), np.float32)
        lse = np.empty((len(heads), L), np.float32)
        vis = C.c_uint64(0)
        secs = self._fn("pipeline_threads")(_ptr(q), _ptr(k), _ptr(v), Z, Hq, Hkv, L, d, B, alpha,
                                            sink_tokens, window_tokens, tau, eps, _ptr(heads),
                                            len(heads), threads, _ptr(out), _ptr(lse),
                                            C.byref(vis))
        if secs < 0:
            raise ValueError("pipeline failed")
        return secs, out, lse, vis.value

    def pipeline_detail(self, q, k, v, B, alpha, sink_tokens, window_tokens, tau, eps, heads,
                        threads, row_keep=None, attend=True):
        """Reference pipeline per (z*Hq + h) slice in `heads`, returning everything the full-size
        parity tests compare (reference shim only).

        row_keep: optional bool[M]; attention runs only on those query-block rows (the other
        rows' counts are zeroed before block_sparse_attention, so their out / lse are NaN / -inf).
        Returns dict(secs, score[n,M,M], idx[n,M,M], counts[n,M], comparisons, out[n,L,d],
        lse[n,L], visits)."""
        f = self._ref_only("pipeline_detail")
        q, k, v = _f(q), _f(k), _f(v)
        Z, Hq, L, d = q.shape
        Hkv = k.shape[1]
        M, _ = self.grid(L, B)
        heads = np.ascontiguousarray(heads, dtype=np.int32)
        n = len(heads)
        keep = None
        if row_keep is not None or not attend:
            keep = np.zeros(M, np.uint8) if not attend else \
                np.ascontiguousarray(row_keep, dtype=np.uint8)
        score = np.empty((n, M, M), np.float32)
        idx = np.empty((n, M, M), np.int32)
        counts = np.empty((n, M), np.int32)
        out = np.empty((n, L, d), np.float32) if attend else None
        lse = np.empty((n, L), np.float32) if attend else None
        cmp, vis = C.c_uint64(0), C.c_uint64(0)
        secs = f(_ptr(q), _ptr(k), _ptr(v), Z, Hq, Hkv, L, d, B, alpha, sink_tokens,
                 window_tokens, tau, eps, _ptr(heads), n, threads, _ptr(keep), _ptr(score),
                 _ptr(idx), _ptr(counts), C.byref(cmp), _ptr(out), _ptr(lse), C.byref(vis))
        if secs < 0:
            raise ValueError("reference pipeline failed")
        return dict(secs=secs, score=score, idx=idx, counts=counts, comparisons=cmp.value,
                    out=out, lse=lse, visits=vis.value)

    # ------------------------------------------------------------------ reference-only (CLI pins)
    def _ref_only(self, name):
        if self.kind != "reference":
            raise NotImplementedError(f"{name}: reference shim only (pins the CLI restatement)")
        return getattr(self.lib, "ref_" + name)

    def generate_alternating_slash(self, strength, offset, noise, seed, Z, H, L, d, B, tau=0.0):
        """workloads.hpp:269-311: returns (q, k, v, ground_truth Z x M x M x H)."""
        f = self._ref_only("generate_alternating_slash")
        f.argtypes = [_f32, _i64, _f32, _u64, _u64, _u64, _u64, _u64, _u32, _f32, _p, _p, _p, _p]
        q = np.empty((Z, H, L, d), np.float32)
        k, v = np.empty_like(q), np.empty_like(q)
        M, _ = self.grid(L, B)
        gt = np.empty((Z, M, M, H), np.uint8)
        self._check(f(strength, offset, noise, seed, Z, H, L, d, B, tau, _ptr(q), _ptr(k), _ptr(v),
                      _ptr(gt)), "generate_alternating_slash")
        return q, k, v, gt

    def heavy_tail_sweep_map(self, n, head_mass, alpha, seed):
        """workloads.hpp:378-399: (score 1 x 1 x n x n, head_index[n])."""
        f = self._ref_only("heavy_tail_sweep_map")
        f.argtypes = [_u32, _f32, _f32, _u64, _p, _p]
        score = np.empty((1, 1, n, n), np.float32)
        head = np.empty(n, np.int32)
        self._check(f(n, head_mass, alpha, seed, _ptr(score), _ptr(head)), "heavy_tail_sweep_map")
        return score, head

    def save_tensor(self, arr, path):
        """tensor.hpp save_tensor (FPT1) for f32 / i32 arrays."""
        arr = np.ascontiguousarray(arr)
        name = "save_tensor_f32" if arr.dtype == np.float32 else "save_tensor_i32"
        f = self._ref_only(name)
        f.argtypes = [_p, _p, _i32, C.c_char_p]
        shape = np.asarray(arr.shape, np.uint64)
        self._check(f(_ptr(arr), _ptr(shape), arr.ndim, os.fsencode(path)), name)

    # ------------------------------------------------------------------ plain numpy helpers
    @staticmethod
    def visit_count(counts) -> int:
        return int(np.asarray(counts, dtype=np.int64).sum())

    @staticmethod
    def density(counts, M: int) -> float:
        Z, _, H = counts.shape
        return Oracle.visit_count(counts) / (Z * H * (M * (M + 1) / 2.0))

    @staticmethod
    def full_causal_plan(Z, H, M):
        idx = np.full((Z, M, M, H), M, np.int32)
        counts = np.empty((Z, M, H), np.int32)
        for i in range(M):
            idx[:, i, : i + 1, :] = np.arange(i + 1, dtype=np.int32)[None, :, None]
            counts[:, i, :] = i + 1
        return idx, counts
