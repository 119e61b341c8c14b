#!/usr/bin/env python
"""Host<->device copy bandwidth with pinned buffers: H2D alone, D2H alone, both concurrently."""
import time

import torch

n = 336 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


a = t(lambda: d.copy_(h, non_blocking=True))
b = t(lambda: h2.copy_(d2, non_blocking=True))
c = t(both)
print(f"H2D {n/a/1e9:.1f} GB/s   D2H {n/b/1e9:.1f} GB/s   concurrent {2*n/c/1e9:.1f} GB/s total")

hh = torch.empty(n, dtype=torch.uint8).pin_memory()
dd = torch.empty(n, dtype=torch.uint8, device="cuda")


def two_in():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        dd.copy_(hh, non_blocking=True)


e = t(two_in)
print(f"two concurrent H2D streams {2*n/e/1e9:.1f} GB/s total")
for mb in (1, 4, 16, 64):
    m = mb << 20
    f = t(lambda: d[:m].copy_(h[:m], non_blocking=True), reps=20)
    g = t(lambda: h2[:m].copy_(d2[:m], non_blocking=True), reps=20)
    print(f"{mb} MiB: H2D {m/f/1e9:.1f} GB/s  D2H {m/g/1e9:.1f} GB/s")
