#!/usr/bin/env python
"""e2e (fpb_host_prefill, pinned host buffers, H2D + kernels + D2H) wall time of the bench
workload; run once per FPB_E2E_CHUNKS setting (read once per process)."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import workload  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = workload.composite(1234, 1, 32, 4, L)
qp, kp, vp = (x.contiguous().pin_memory() for x in (q, k, v))
outp = torch.empty(qp.shape, dtype=torch.bfloat16).pin_memory()
lsep = torch.empty(qp.shape[:3], dtype=torch.float32).pin_memory()
cfg = fp.PipelineConfig()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(8):
    flush.fill_(3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
    if i >= 2:
        ts.append((time.perf_counter() - t0) * 1e3)
print(f"chunks={os.environ.get('FPB_E2E_CHUNKS', 'default')} L={L} e2e ms median "
      f"{statistics.median(ts):.3f} min {min(ts):.3f}")
