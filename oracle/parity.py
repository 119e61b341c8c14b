"""Full-size parity checks of the GPU path against the reference pipeline — TEST INFRASTRUCTURE.

Used by tests/test_gpu_fullsize_parity.py and by bench.py's cpu_baseline leg (which already runs
the unmodified reference on sampled Q heads of the bench workload and compares its plan and
output with the GPU step's).  The bars are north_star's:

* masks / idx / counts: bit-exact, except blocks whose reference score lies within
  MASK_EPS * thresh of the row threshold (selection.hpp:75-84); those are counted ("near") and
  the number that actually differ is reported ("flipped");
* attention out and lse (base 2): max-abs <= 2e-2 and mean-abs <= 1e-3 against the reference's
  fp32 result (attention.hpp:38-132), compared on the rows whose GPU plan row equals the
  reference's bit for bit (a near-threshold flip changes the visited blocks, so such a row has no
  same-plan reference).
"""
from __future__ import annotations

import numpy as np

OUT_MAX_ABS = 2e-2
OUT_MEAN_ABS = 1e-3
MASK_EPS = 1e-4


def plan_to_mask(idx: np.ndarray, counts: np.ndarray) -> np.ndarray:
    """Per-slice plan (n x M x N idx, n x M counts) -> n x M x N bool mask (compress_indices
    inverse, selection.hpp:176-192).  Validates the plan invariants on the way: strictly
    increasing active prefix, fill value N after it."""
    n, M, N = idx.shape
    slot = np.arange(N)[None, None, :]
    live = slot < counts[:, :, None]
    if not np.all(idx[~live] == N):
        raise AssertionError("plan slots past the count must hold the fill value N")
    inc = (idx[:, :, 1:] > idx[:, :, :-1]) | ~live[:, :, 1:]
    if not np.all(inc):
        raise AssertionError("active plan prefix must be strictly increasing")
    mask = np.zeros((n, M, N + 1), bool)
    nn, ii, _ = np.nonzero(live)
    mask[nn, ii, idx[live]] = True
    return mask[:, :, :N]


def near_band(score: np.ndarray, alpha: float, eps: float = MASK_EPS) -> np.ndarray:
    """n x M x N bool: causal blocks whose reference score is within eps*thresh of
    thresh = alpha * max(0, causal row max) (selection.hpp:75-80)."""
    n, M, N = score.shape
    tri = np.tril(np.ones((M, N), bool))[None]
    s = np.where(tri, score, np.float32(0))
    th = (np.float32(alpha) * np.maximum(s.max(axis=2), 0).astype(np.float32))[..., None]
    return tri & (np.abs(score - th) <= eps * th)


def compare_plans(gpu_idx, gpu_counts, ref_idx, ref_counts, ref_score, alpha,
                  eps: float = MASK_EPS) -> dict:
    """All arrays per slice: idx n x M x N, counts n x M, score n x M x N."""
    gm = plan_to_mask(gpu_idx, gpu_counts)
    rm = plan_to_mask(ref_idx, ref_counts)
    near = near_band(ref_score, alpha, eps)
    diff = gm != rm
    same_row = np.all(gpu_idx == ref_idx, axis=2) & (gpu_counts == ref_counts)
    near_rows = near.any(axis=2)
    return {
        "blocks": int(np.tril(np.ones(ref_score.shape[1:], bool)).sum()) * ref_score.shape[0],
        "mismatch_outside_band": int((diff & ~near).sum()),
        "near": int(near.sum()),
        "flipped": int((diff & near).sum()),
        "rows": int(same_row.size),
        "rows_identical": int(same_row.sum()),
        # rows without any near-threshold block must be bit-identical (idx and counts)
        "rows_differ_without_near": int((~same_row & ~near_rows).sum()),
        "same_row": same_row,
    }


def compare_outputs(gpu_out, gpu_lse, ref_out, ref_lse, rows_ok, block: int) -> dict:
    """gpu/ref out n x L x d, lse n x L (base 2); rows_ok n x M bool = query blocks to compare."""
    n, L = ref_lse.shape
    tok = np.repeat(rows_ok, block, axis=1)[:, :L]
    if not tok.any():
        return {"tokens": 0, "out_max": 0.0, "out_mean": 0.0, "lse_max": 0.0, "lse_mean": 0.0}
    do = np.abs(np.asarray(gpu_out, np.float64)[tok] - np.asarray(ref_out, np.float64)[tok])
    dl = np.abs(np.asarray(gpu_lse, np.float64)[tok] - np.asarray(ref_lse, np.float64)[tok])
    return {"tokens": int(tok.sum()), "out_max": float(do.max()), "out_mean": float(do.mean()),
            "lse_max": float(dl.max()), "lse_mean": float(dl.mean())}


def within_bars(po: dict, pp: dict) -> bool:
    return (pp["mismatch_outside_band"] == 0 and pp["rows_differ_without_near"] == 0
            and po["out_max"] <= OUT_MAX_ABS and po["out_mean"] <= OUT_MEAN_ABS
            and po["lse_max"] <= OUT_MAX_ABS and po["lse_mean"] <= OUT_MEAN_ABS)
