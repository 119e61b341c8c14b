"""Golden vectors for the CLI front-end, produced by the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):  python tests/golden/gen_cli_golden.py
Pins the CLI's own restatements (tools/cli/workloads.hpp, include/fpb200/fpt1.hpp) against the
reference's generate_alternating_slash (workloads.hpp:269-311), heavy_tail_sweep_map
(workloads.hpp:378-399) and save_tensor (tensor.hpp FPT1 writer).  tests/test_cli.py consumes it.
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Oracle  # noqa: E402

# alt-slash: (strength, offset, noise, seed, Z, H, L, d, B)
ALT = (2.5, 128, 0.5, 5, 1, 1, 384, 16, 64)
# heavy-tail sweep map: the reference CLI test's case (L 8192, B 128 -> n 64; alpha fixed 0.2)
HEAVY = (64, 0.7, 0.2, 6)


def main():
    R = Oracle("reference")
    out = {"alt_params": np.array(ALT, np.float64), "heavy_params": np.array(HEAVY, np.float64)}
    s, off, noise, seed, Z, H, L, d, B = ALT
    tau = 1.0 / np.sqrt(np.float32(d))
    q, k, v, gt = R.generate_alternating_slash(s, off, noise, seed, Z, H, L, d, B, float(tau))
    out.update(alt_q=q, alt_k=k, alt_v=v, alt_gt=gt)
    score, head = R.heavy_tail_sweep_map(*HEAVY)
    out.update(heavy_score=score, heavy_head=head)
    rng = np.random.default_rng(0)
    f32 = rng.standard_normal((2, 3, 5)).astype(np.float32)
    i32 = rng.integers(-5, 100, (1, 4, 2), dtype=np.int32)
    with tempfile.TemporaryDirectory() as tmp:
        for name, arr in (("f32", f32), ("i32", i32)):
            p = os.path.join(tmp, name + ".fpt")
            R.save_tensor(arr, p)
            out[f"fpt_{name}_array"] = arr
            out[f"fpt_{name}_bytes"] = np.frombuffer(open(p, "rb").read(), np.uint8)
    path = os.path.join(HERE, "cli.npz")
    np.savez_compressed(path, **out)
    print(f"cli.npz -> {os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
