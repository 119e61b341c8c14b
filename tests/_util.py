"""Shared helpers for the parity tests (inputs, tolerances, epsilon-band mask comparison)."""
from __future__ import annotations

import numpy as np

# north_star / SURVEY §8c tolerances
OUT_MAX_ABS = 2e-2
OUT_MEAN_ABS = 1e-3
MASK_EPS = 1e-4  # relative band around alpha * max_ref in which a mask bit may differ


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as the exact fp32 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def thresholds(score: np.ndarray, alpha: float) -> np.ndarray:
    """alpha * max(0, causal row max) per (z, h, i) — selection.hpp:75-80."""
    Z, H, M, N = score.shape
    tri = np.tril(np.ones((M, N), bool))
    s = np.where(tri[None, None], score, 0.0)
    return (np.float32(alpha) * np.maximum(s.max(axis=3), 0).astype(np.float32)).astype(np.float32)


def near_threshold(score_ref: np.ndarray, alpha: float, eps: float = MASK_EPS) -> np.ndarray:
    """Z x H x M x N bool: causal blocks whose reference score lies within eps*thresh of thresh."""
    th = thresholds(score_ref, alpha)[..., None]
    M = score_ref.shape[2]
    tri = np.tril(np.ones((M, M), bool))[None, None]
    return tri & (np.abs(score_ref - th) <= eps * th)


def compare_masks(mask_gpu: np.ndarray, mask_ref: np.ndarray, score_ref: np.ndarray,
                  alpha: float, eps: float = MASK_EPS):
    """Masks are Z x M x N x H.  Returns (n_mismatch_outside_band, n_near, n_mismatch_in_band)."""
    near = near_threshold(score_ref, alpha, eps).transpose(0, 2, 3, 1)  # -> Z x M x N x H
    diff = mask_gpu != mask_ref
    return int((diff & ~near).sum()), int(near.sum()), int((diff & near).sum())


def rows_with_near(score_ref, alpha, eps=MASK_EPS) -> np.ndarray:
    """Z x M x H bool: plan rows containing at least one near-threshold block."""
    return near_threshold(score_ref, alpha, eps).any(axis=3).transpose(0, 2, 1)


def err(a: np.ndarray, b: np.ndarray):
    d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    return float(d.max()), float(d.mean())


def composite_np(seed: int, Z: int, Hq: int, Hkv: int, L: int, d: int = 128, B: int = 128,
                 noise: float = 0.5, n_vertical: int = 4, n_slash: int = 2):
    """Small vertical+slash workload in numpy (fp32), for oracle-sized parity cases."""
    rng = np.random.default_rng(seed)
    tau = 1.0 / np.sqrt(d)
    M = (L + B - 1) // B
    q = rng.normal(0, noise, (Z, Hq, L, d)).astype(np.float32)
    k = rng.normal(0, noise, (Z, Hkv, L, d)).astype(np.float32)
    v = rng.normal(0, noise, (Z, Hkv, L, d)).astype(np.float32)
    g = Hq // Hkv
    for z in range(Z):
        for kh in range(Hkv):
            for _ in range(n_vertical):
                col = rng.integers(0, M)
                u = rng.normal(size=d)
                u /= np.linalg.norm(u)
                k[z, kh, col * B:(col + 1) * B] += (np.sqrt(n_vertical) * u).astype(np.float32)
                for hq in range(kh * g, (kh + 1) * g):
                    s = rng.uniform(0.5, 3.0)
                    q[z, hq] += (s / tau / np.sqrt(n_vertical) * u).astype(np.float32)
            for _ in range(n_slash):
                off = int(rng.integers(1, max(2, L // 4)))
                dirs = rng.normal(size=(M, d))
                dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
                tok = np.arange(L) // B
                if off < L:
                    k[z, kh, : L - off] += dirs[tok[off:]].astype(np.float32)
                for hq in range(kh * g, (kh + 1) * g):
                    s = rng.uniform(0.5, 3.0)
                    q[z, hq] += (s / tau / np.sqrt(max(1, n_slash)) * dirs[tok]).astype(np.float32)
    return q, k, v


# ------------------------------------------------------------------ FPT1 container (tensor.hpp:97-221)
_FPT_DTYPES = {0: np.float32, 1: np.int32}


def write_fpt(path, arr) -> None:
    """Little-endian FPT1: magic, u32 version 1, u32 ndim, u64 dims, u32 dtype (0 f32 / 1 i32)."""
    arr = np.ascontiguousarray(arr)
    code = {np.dtype(np.float32): 0, np.dtype(np.int32): 1}[arr.dtype]
    hdr = b"FPT1" + np.array([1, arr.ndim], "<u4").tobytes() + np.array(arr.shape, "<u8").tobytes()
    with open(path, "wb") as f:
        f.write(hdr + np.array([code], "<u4").tobytes() + arr.astype(arr.dtype.newbyteorder("<")).tobytes())


def read_fpt(path) -> np.ndarray:
    raw = open(path, "rb").read()
    assert raw[:4] == b"FPT1", "bad magic"
    version, ndim = np.frombuffer(raw, "<u4", 2, 4)
    assert version == 1
    shape = tuple(int(x) for x in np.frombuffer(raw, "<u8", int(ndim), 12))
    off = 12 + 8 * int(ndim)
    code = int(np.frombuffer(raw, "<u4", 1, off)[0])
    n = int(np.prod(shape))
    data = np.frombuffer(raw, np.dtype(_FPT_DTYPES[code]).newbyteorder("<"), n, off + 4)
    assert off + 4 + 4 * n == len(raw), "trailing bytes"
    return data.reshape(shape).astype(_FPT_DTYPES[code])
