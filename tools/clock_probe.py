#!/usr/bin/env python
"""SM clock / power while the attention kernel runs back to back at a given length (NVML)."""
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06199_b200 as fp  # noqa: E402
from paper_2603_06199_b200 import workload  # noqa: E402
import pynvml  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
q, k, v = workload.composite(5, 1, 32, 4, L, device="cuda")
cfg = fp.PipelineConfig()
r = fp.PrefillRunner(q, k, v, cfg).capture()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for _ in range(3):
    r.replay_discover()
    r.replay_attend()
torch.cuda.synchronize()
clk, pw = [], []
t0 = time.time()
n = 0
while time.time() - t0 < 3.0:
    r.replay_attend()
    n += 1
    if n % 2 == 0:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
        torch.cuda.synchronize()
clk.sort()
pw.sort()
reasons = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
print(f"L={L}: sm clock median {clk[len(clk)//2]} MHz (min {clk[0]}, max {clk[-1]}), "
      f"power median {pw[len(pw)//2]:.0f} W (max {pw[-1]:.0f}), throttle reasons 0x{reasons:x}")
