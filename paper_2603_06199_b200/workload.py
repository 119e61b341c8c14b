"""Synthetic FlashPrefill inputs: graded vertical + slash patterns planted in Q/K geometry.

The reference only has single-pattern generators (workloads.hpp:149-263); the composite used by
bench.py and the large parity cases follows the same logit-geometry construction:
background N(0, noise^2); per KV head, `n_vertical` key blocks receive sqrt(n_v) * u and every Q
head of the group adds (s / tau / sqrt(n_v)) * u with s ~ U(smin, smax) per head; `n_slash` slash
offsets ~ U(1, L/4) are realised like workloads.hpp:187-209 (query row t and key row t - offset
share the direction of t's block).  Generation runs on the CPU with a seeded torch.Generator so
the GPU arm and the CPU reference arm of bench.py see byte-identical inputs.
"""
from __future__ import annotations

import math

import torch


def composite(seed: int, Z: int, Hq: int, Hkv: int, L: int, d: int = 128, B: int = 128,
              noise: float = 0.5, n_vertical: int = 8, n_slash: int = 4, smin: float = 0.5,
              smax: float = 3.0, dtype: torch.dtype = torch.bfloat16, device: str = "cpu"):
    """Returns tensors (q, k, v) of shapes Z x Hq x L x d and Z x Hkv x L x d in `dtype`.

    device="cpu" (default) is reproducible across machines; device="cuda" is for very long
    sequences (same recipe, different random stream)."""
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    g = torch.Generator(device=device).manual_seed(seed)
    tau = 1.0 / math.sqrt(d)
    M = (L + B - 1) // B
    kw = dict(generator=g, device=device)
    q = torch.randn((Z, Hq, L, d), **kw).mul_(noise)
    k = torch.randn((Z, Hkv, L, d), **kw).mul_(noise)
    v = torch.randn((Z, Hkv, L, d), **kw).mul_(noise)
    grp = Hq // Hkv
    blk = torch.arange(L, device=device) // B
    for z in range(Z):
        for kh in range(Hkv):
            heads = range(kh * grp, (kh + 1) * grp)
            if n_vertical > 0:
                cols = torch.randint(0, M, (n_vertical,), **kw)
                u = torch.randn((n_vertical, d), **kw)
                u /= u.norm(dim=1, keepdim=True)
                for i in range(n_vertical):
                    c = int(cols[i])
                    k[z, kh, c * B:min(L, (c + 1) * B)] += math.sqrt(n_vertical) * u[i]
                for h in heads:
                    s = torch.empty(n_vertical, device=device).uniform_(smin, smax, generator=g)
                    q[z, h] += (s / tau / math.sqrt(n_vertical)) @ u
            for _ in range(n_slash):
                off = int(torch.randint(1, max(2, L // 4), (1,), **kw))
                dirs = torch.randn((M, d), **kw)
                dirs /= dirs.norm(dim=1, keepdim=True)
                rows = dirs[blk]  # L x d: direction of each token's block
                if off < L:
                    k[z, kh, : L - off] += rows[off:]
                for h in heads:
                    s = float(torch.empty(1, device=device).uniform_(smin, smax, generator=g))
                    q[z, h] += (s / tau / math.sqrt(n_slash)) * rows
    return q.to(dtype).contiguous(), k.to(dtype).contiguous(), v.to(dtype).contiguous()


def qwen3_30b_a3b(L: int, Z: int = 1, seed: int = 0, dtype=torch.bfloat16, device="cpu"):
    """Qwen3-30B-A3B attention layer shape: 32 Q heads, 4 KV heads, d = 128."""
    return composite(seed, Z, 32, 4, L, dtype=dtype, device=device)


def llama31_8b(L: int, Z: int = 1, seed: int = 0, dtype=torch.bfloat16, device="cpu"):
    """Llama-3.1-8B attention layer shape: 32 Q heads, 8 KV heads, d = 128."""
    return composite(seed, Z, 32, 8, L, dtype=dtype, device=device)
