"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref/libbsattn_ref.so).

Run in the build container (where /root/reference exists):  python tests/golden/gen_golden.py
Each case records how its inputs are produced (the reference's own generate_planted /
random_batch recipes, restated bit-exactly by oracle/bsattn_oracle.c) plus the reference outputs,
so the fixtures stay small.  tests/test_oracle_golden.py pins the C restatement against them and
tests/test_gpu_parity.py::test_golden_* pins the CUDA path against them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Oracle  # noqa: E402
from tests._util import bf16_round  # noqa: E402

# (name, kind, strength, a, b, noise, seed, Z, H, L, d, B, bf16)
CASES = [
    ("vertical_L1000_d32", 0, 2.5, 3, 0, 0.5, 1, 1, 2, 1000, 32, 128, False),
    ("slash_L2048_d32", 1, 2.5, 300, 0, 0.5, 2, 1, 2, 2048, 32, 128, False),
    ("block_L777_B64_d16", 2, 5.0, 9, 4, 1.0, 3, 2, 1, 777, 16, 64, False),
    ("needle_L1500_d32", 3, 2.5, 1234, 0, 0.5, 4, 1, 1, 1500, 32, 128, False),
    # d = 128, B = 128, bf16-exact inputs: consumed by the GPU golden tests
    ("gpu_slash_L1024_d128", 1, 2.5, 200, 0, 0.5, 5, 1, 2, 1024, 128, 128, True),
    ("gpu_vertical_L1300_d128", 0, 2.5, 2, 0, 0.5, 6, 1, 2, 1300, 128, 128, True),
]
ALPHAS = [0.0, 0.12, 0.5]


def inputs(o: Oracle, case):
    name, kind, strength, a, b, noise, seed, Z, H, L, d, B, bf = case
    q, k, v, gt = o.generate_planted(kind, strength, a, b, noise, seed, Z, H, L, d, B)
    if bf:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v, gt


def main():
    R = Oracle("reference")
    for case in CASES:
        name, kind, strength, a, b, noise, seed, Z, H, L, d, B, bf = case
        q, k, v, gt = inputs(R, case)
        tau = float(R.scale(d))
        M = (L + B - 1) // B
        out = {"params": np.array([kind, strength, a, b, noise, seed, Z, H, L, d, B, int(bf)],
                                  dtype=np.float64),
               "gt": gt, "pooled": R.pool_keys(k, B)}
        en, lm, sc = R.discover(q, k, B, tau)
        out.update(energy=en, local_max=lm, score=sc)
        for al in ALPHAS:
            mask, cmp = R.max_threshold_mask(sc, B, al, 256, 512)
            idx, counts = R.compress_indices(mask)
            tag = f"a{int(al * 100):03d}"
            out[f"mask_{tag}"] = mask
            out[f"cmp_{tag}"] = np.array([cmp], np.uint64)
            out[f"idx_{tag}"] = idx
            out[f"counts_{tag}"] = counts
            if al == 0.12:
                o, lse, vis = R.block_sparse_attention(q, k, v, idx, counts, B, tau)
                out.update(out_sparse=o, lse_sparse=lse, visits=np.array([vis], np.uint64))
        if not bf:  # comparison baselines (selection.hpp:94-159, discovery.hpp:161-279)
            out["topk4"] = R.sort_select(sc, "topk", 4, B, 256, 512)
            out["topp09"] = R.sort_select(sc, "topp", 0.9, B, 256, 512)
            for method in ("pool-both", "exact"):
                e2, l2, s2 = R.discover_variant(method, q, k, B, tau)
                tag = method.replace("-", "_")
                out.update({f"{tag}_energy": e2, f"{tag}_local_max": l2, f"{tag}_score": s2})
        if L <= 1100:
            o, lse = R.dense_attention(q, k, v, tau)
            out.update(out_dense=o, lse_dense=lse)
        # hashes of the generated inputs (pins the restated generator, not just the outputs)
        out["q_sum"] = np.array([q.astype(np.float64).sum(), k.astype(np.float64).sum(),
                                 v.astype(np.float64).sum()])
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: M={M} -> {os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
