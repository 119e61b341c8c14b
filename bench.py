#!/usr/bin/env python
"""FlashPrefill B200 benchmark — sparse-prefill attention on the Qwen3-30B-A3B layer shape.

One step = the whole FlashPrefill hot path over ONE synthetic Qwen3 layer resident in HBM:
  fpb_discover_select (K1 pooling inside the K2/K3 tcgen05 discovery launch, threshold, compaction)
  -> fpb_block_sparse_attention (K4 tcgen05 block-sparse FlashAttention)
  -> (N > 1) the all-gather of O and LSE across ranks (NCCL), inside the timed region.
Metric: effective TFLOP/s = dense-causal-equivalent FLOPs 4*d*Z*Hq*L(L+1)/2 of the layer / step
time, max over ranks; ms_per_step is reported beside it.

  python bench.py [--gpus N --steps K --warmup W] [--impl fpb200|reference] [--L 32768]
                  [--partition kv|kv_zigzag|rows|zigzag]
  N > 1 (torchrun, one rank per GPU): strong scaling of the one layer.  `kv` (default, north_star)
  gives rank g a KV-head group (kv_group_shard; with N > Hkv a group's Q heads are split and its
  KV head replicated); `kv_zigzag` keeps one KV head per rank but splits a group's rows (zigzag)
  instead of its Q heads; `rows` / `zigzag` give every rank a share of every head's query blocks.
  No collective inside the kernels; one all-gather of O + LSE after them.

L2 hygiene: a 512 MiB buffer is written between timed steps (L2 is 126 MB); each step is timed
with CUDA events on the launching stream; max over ranks.  N = 1 also emits `sweep` (4K / 32K /
128K / 256K, device-resident, same recipe) and the reference comparison `parity`.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "sparse prefill attention ms & TFLOP/s/GPU at 4K–256K, Qwen3-30B-A3B shape"
UNIT = "TFLOP/s (effective, dense-causal-equivalent)"
B = 128
D = 128
SWEEP_LS = (4096, 32768, 131072, 262144)


def peaks():
    try:
        with open(MEASURED) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "tc_burst": p["bf16_tflops"],
                "tc_sustained": p["bf16_tflops_sustained"], "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "tc_burst": 1590.0, "tc_sustained": 1400.0, "src": "fallback"}


def ncu_traffic(kernel: str, cfg: dict):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of `kernel` from the
    committed `ncu --set full` captures (profiles/ncu_traffic.json, written by
    tools/ncu_summary.py --traffic, one record per captured config); None unless a capture was
    taken on this exact config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            recs = json.load(f)[kernel]
    except (OSError, KeyError, ValueError):
        return None
    for rec in recs if isinstance(recs, list) else [recs]:
        if all(rec.get("config", {}).get(k) == v for k, v in cfg.items()):
            return rec["dram_bytes"]
    return None


class ClockSampler:
    """SM clocks / throttle reasons sampled via NVML every ~2 ms DURING the timed region
    (nvidia-smi's 200 ms loop is too coarse for a ~20 ms region)."""

    REASONS = {  # nvmlClocksEventReason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml, 2 ms poll during the timed steps"}


def dense_flops(Z, Hq, L):
    return 4.0 * D * Z * Hq * L * (L + 1) / 2.0


def plan_flops(counts: torch.Tensor, idx: torch.Tensor, rows=None):
    """Algorithmic FLOPs of the visited blocks: 4 d B^2 off-diagonal, 4 d B(B+1)/2
    on the diagonal.  rows: optional list of the query blocks this plan owns (row shards leave
    the other rows unwritten)."""
    Z, M, H = counts.shape
    ar = torch.arange(M, device=idx.device)
    own = torch.zeros(M, dtype=torch.bool, device=idx.device)
    own[torch.as_tensor(rows, device=idx.device) if rows is not None else ar] = True
    c = torch.where(own.view(1, M, 1), counts, torch.zeros_like(counts)).to(torch.int64)
    visits = int(c.sum())
    slot = ar.view(1, 1, M, 1)
    within = slot < c.view(Z, M, 1, H)
    diag = int(((idx == ar.view(1, M, 1, 1)) & within).sum())
    f = 4.0 * D * ((visits - diag) * B * B + diag * B * (B + 1) / 2.0)
    return f, visits, diag


def make_inputs(args):
    """The one synthetic layer every rank (and the reference arm) sees: generated on the CPU from
    a fixed seed, so all arms get byte-identical tensors."""
    from paper_2603_06199_b200 import workload
    return workload.composite(args.seed, 1, args.hq, args.hkv, args.L,
                              n_vertical=args.n_vertical, n_slash=args.n_slash)


def bench_config(args, world):
    """The `config` object — identical in both arms (the driver compares them)."""
    part = {"kv": "KV-head-group shards (kv_group_shard)",
            "rows": "interleaved query-block shards (fpb_*_rows)",
            "zigzag": "zigzag query-block shards (fpb_*_zigzag)",
            "kv_zigzag": "KV-head-group shards, a group's ranks split by zigzag query-block "
                         "chunks (kv_zigzag_shard)"}[args.partition]
    return {"workload": f"Qwen3-30B-A3B attention layer (Hq={args.hq}, Hkv={args.hkv}, d=128) "
                        f"bf16 causal L={args.L}, alpha={args.alpha}, B=128, sink 256, window 512",
            "global_batch_sequences": 1, "seq_len": args.L,
            "parallelism": (f"one layer split over {world} GPU(s): {part}; NCCL gather of "
                            f"O + LSE inside the timed step"
                            + (f", overlapped with compute in {args.gather_chunks} head chunks"
                               if args.partition == "kv" and args.gather_chunks > 1 else "")
                            if world > 1 else "1 GPU"),
            "l2": "512 MiB buffer written between timed steps (L2 126 MB)",
            "seed": args.seed}


# ------------------------------------------------------------------------------ CPU reference
def sample_heads(Hq: int, Hkv: int, n: int) -> list[int]:
    """Spread the sample over KV groups: head order 0, g, 2g, ..., 1, g+1, ..."""
    g = Hq // Hkv
    order = [kh * g + j for j in range(g) for kh in range(Hkv)]
    return order[:max(1, min(n, Hq))]


def reference_pipeline(q, k, v, args, threads: int, heads: list[int]):
    """The reference pipeline (oracle/_ref = the unmodified reference headers; the C port if the
    reference was not built) on the given (z*Hq + h) slices: discover -> max_threshold_mask ->
    compress_indices -> block_sparse_attention (acceptance.cpp:357-360), one slice per thread.
    Returns (result dict or None, kind)."""
    from oracle import Oracle, available
    tau = float(1.0 / math.sqrt(D))
    if available("reference"):
        r = Oracle("reference").pipeline_detail(q, k, v, B, args.alpha, 256, 512, tau, 1e-10,
                                                heads, threads)
        return r, "reference"
    secs, out, lse, visits = Oracle("port").pipeline(q, k, v, B, args.alpha, 256, 512, tau,
                                                     1e-10, heads, threads)
    return {"secs": secs, "out": out, "lse": lse, "visits": visits}, "port"


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    q, k, v = make_inputs(args)
    qf, kf, vf = (x.float().numpy() for x in (q, k, v))
    heads = sample_heads(args.hq, args.hkv, args.ref_heads or threads)
    times = []
    kind = None
    for i in range(args.warmup + args.steps):
        r, kind = reference_pipeline(qf, kf, vf, args, threads, heads)
        if i >= args.warmup:
            times.append(r["secs"])
    t = statistics.mean(times)
    value = dense_flops(1, len(heads), args.L) / t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (vertical+slash composite planted in Q/K geometry, seeded; bf16 values "
                "upcast exactly to fp32)",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{len(heads)} of {args.hq} Q heads of the layer per step (one "
                                   f"per thread), full L={args.L}, discover->mask->compress->"
                                   f"sparse attention per head; value normalised per head"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def _coll_device(dist, dev):
    return torch.device("cpu") if dist.get_backend() == "gloo" else dev


def owned_rows(args, M, world, rank):
    from paper_2603_06199_b200 import shard
    if args.partition == "rows" and world > 1:
        return list(range(rank, M, world))
    if args.partition == "zigzag" and world > 1:
        return shard.zigzag_blocks(M, world, rank)
    if args.partition == "kv_zigzag" and world > 1:
        _, rows = shard.kv_zigzag_shard(args.hq, args.hkv, world, rank,
                                        getattr(args, "kv_weights_used", None))
        return None if rows is None else shard.zigzag_blocks(M, rows[2], rows[1])
    return None


class ChunkedKvStep:
    """A KV-group shard computed as `chunks` chunks of its Q heads (each its own PrefillRunner over
    the shared K/V), each chunk's O / LSE sent to every peer while the next chunk computes
    (shard.OverlappedHeadGather: NCCL point-to-point into the final layout)."""

    def __init__(self, fp, shard, args, q, k, v, cfg, s, chunks):
        ql, kl, vl = shard.local_slices(q, k, v, s)
        self.ranges = shard.head_chunks(s.hq, chunks)
        self.runners = [fp.PrefillRunner(ql[:, a:b].contiguous(), kl, vl, cfg,
                                         out_dtype=torch.bfloat16) for a, b in self.ranges]
        self.out = torch.empty(q.shape, dtype=torch.bfloat16, device=q.device)
        self.lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
        self.gather = shard.OverlappedHeadGather(args.hq, args.hkv, self.out, self.lse)

    def capture(self):
        for r in self.runners:
            r.capture()
        return self

    @property
    def graphs(self):
        return [g for r in self.runners for g in r.graphs]

    def check(self):
        return sum(r.check() for r in self.runners)

    def plans(self):
        return [(r.counts, r.idx) for r in self.runners]

    def step(self, stream=None, marks=None):
        """One step; marks (list) collects (discover-end, attend-end) events per chunk."""
        for (a, b), r in zip(self.ranges, self.runners):
            r.replay_discover()
            if marks is not None:
                marks.append(torch.cuda.Event(enable_timing=True))
                marks[-1].record(stream)
            r.replay_attend()
            if marks is not None:
                marks.append(torch.cuda.Event(enable_timing=True))
                marks[-1].record(stream)
            self.gather.post(a, b, r.out, r.lse)
        self.gather.wait()


def kv_weights(fp, args, q, k, cfg, world):
    """Per-KV-group work weights for --partition kv_zigzag --kv-weights plan: block visits of each
    group's Q heads from one calibration discovery of the layer (outside the timed region; the
    same on every rank: same inputs, deterministic plan).  None = equal ranks per group."""
    if args.kv_weights != "plan" or world <= args.hkv:
        return None  # at most one rank per group: nothing to weigh
    plan = fp.discover_select(q, k, cfg)[0]
    per_head = plan.counts.sum(dim=(0, 1)).double()  # Z x M x Hq -> per Q head
    g = args.hq // args.hkv
    w = [float(per_head[i * g:(i + 1) * g].sum()) for i in range(args.hkv)]
    args.kv_weights_used = w
    del plan
    return w


def make_runner(fp, args, q, k, v, cfg, world, rank):
    """This rank's PrefillRunner (its shard of the layer) and a gather closure."""
    from paper_2603_06199_b200 import shard
    if world == 1:
        return fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16), None, (0, args.hq)
    if args.partition == "kv" and args.gather_chunks > 1 and q.shape[0] == 1:
        s = shard.kv_group_shard(args.hq, args.hkv, world, rank)
        return (ChunkedKvStep(fp, shard, args, q, k, v, cfg, s, args.gather_chunks), None,
                (s.q_lo, s.q_hi))
    if args.partition == "kv_zigzag":
        w = kv_weights(fp, args, q, k, cfg, world)
        s, rows = shard.kv_zigzag_shard(args.hq, args.hkv, world, rank, w)
        ql, kl, vl = shard.local_slices(q, k, v, s)
        r = fp.PrefillRunner(ql, kl, vl, cfg, out_dtype=torch.bfloat16, rows=rows)
        out_full = torch.empty(q.shape, dtype=torch.bfloat16, device=q.device)
        lse_full = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
        return r, lambda: shard.gather_kv_zigzag(r.out, r.lse, args.hq, args.hkv, B,
                                                 out=out_full, lse=lse_full,
                                                 weights=w), (s.q_lo, s.q_hi)
    if args.partition == "kv":
        s = shard.kv_group_shard(args.hq, args.hkv, world, rank)
        ql, kl, vl = shard.local_slices(q, k, v, s)
        r = fp.PrefillRunner(ql, kl, vl, cfg, out_dtype=torch.bfloat16)
        out_full = torch.empty(q.shape, dtype=torch.bfloat16, device=q.device)
        lse_full = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
        return r, lambda: shard.gather_heads(r.out, r.lse, args.hq, args.hkv,
                                             out=out_full, lse=lse_full), (s.q_lo, s.q_hi)
    rows = shard.row_shard(world, rank) if args.partition == "rows" \
        else shard.zigzag_shard(world, rank)
    r = fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16, rows=rows)
    g = shard.gather_rows if args.partition == "rows" else shard.gather_zigzag
    return r, lambda: g(r.out, r.lse, B), (0, args.hq)


def do_step(runner, gather=None):
    if isinstance(runner, ChunkedKvStep):
        runner.step()
        return
    runner.replay_discover()
    runner.replay_attend()
    if gather:
        gather()


def plan_totals(runner, rows):
    """(algorithmic FLOPs, visits, diagonal visits) of this rank's plan(s)."""
    plans = runner.plans() if isinstance(runner, ChunkedKvStep) else [(runner.counts, runner.idx)]
    tot = [0.0, 0, 0]
    for counts, idx in plans:
        f, vis, diag = plan_flops(counts, idx, rows)
        tot = [tot[0] + f, tot[1] + vis, tot[2] + diag]
    return tot


def time_runner(runner, stream, flush, reps, gather=None, dist=None):
    """CUDA-event times (ms lists) of discover, attend, gather and the whole step, L2 flushed
    between steps.  For a ChunkedKvStep, discover / attend are summed over the chunks and
    `gather` is the exposed part of the transfers (step minus compute)."""
    ts = {"step": [], "disc": [], "attn": [], "gather": []}
    if isinstance(runner, ChunkedKvStep):
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if dist:
                dist.barrier()
            marks = []
            e0.record(stream)
            runner.step(stream, marks)
            e1.record(stream)
            torch.cuda.synchronize()
            starts = [e0] + marks[1::2][:-1]
            disc = sum(a.elapsed_time(b) for a, b in zip(starts, marks[0::2]))
            attn = sum(a.elapsed_time(b) for a, b in zip(marks[0::2], marks[1::2]))
            step = e0.elapsed_time(e1)
            ts["step"].append(step)
            ts["disc"].append(disc)
            ts["attn"].append(attn)
            ts["gather"].append(step - disc - attn)
        return ts
    for _ in range(reps):
        flush.fill_(1)  # evict L2 between steps (not timed)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if dist:
            dist.barrier()
        ev[0].record(stream)
        runner.replay_discover()
        ev[1].record(stream)
        runner.replay_attend()
        ev[2].record(stream)
        if gather:
            gather()
        ev[3].record(stream)
        torch.cuda.synchronize()
        ts["step"].append(ev[0].elapsed_time(ev[3]))
        ts["disc"].append(ev[0].elapsed_time(ev[1]))
        ts["attn"].append(ev[1].elapsed_time(ev[2]))
        ts["gather"].append(ev[2].elapsed_time(ev[3]))
    return ts


def discovery_tensor_view(args, M, ms_disc, pk):
    """The discovery stage against the tensor pipe, its binding resource at <= 128K (the HBM view
    above is what north_star asks for).  Executed MMA FLOPs: per (z, h, query block I) one UMMA
    per 128-block chunk of key blocks J <= I, two of them (k̄ hi and lo, 128 x 128 x 128 each), an
    M = 64 UMMA (half) for a last chunk with <= 64 causal key blocks (csrc/discover.cu).
    Algorithmic FLOPs: 2 d per (query row, causal key block) — the block-approximate logits once."""
    full = half = 0
    for I in range(M):
        n = I // B + 1
        if I % B < 64:
            full += n - 1
            half += 1
        else:
            full += n
    per_head_mma = 2 * (full + 0.5 * half) * 2.0 * B * B * D
    executed = per_head_mma * args.hq / (ms_disc * 1e-3) / 1e12
    algorithmic = args.hq * B * (M * (M + 1) / 2) * 2.0 * D / (ms_disc * 1e-3) / 1e12
    return {"executed_tflops": executed, "frac_of_burst": executed / pk["tc_burst"],
            "algorithmic_tflops": algorithmic,
            "note": "stage time (pooling + discovery + select) in the denominator; executed = "
                    "split-precision UMMAs incl. chunk padding, 2.5x the algorithmic logits"}


def kernel_launches(runner, fallback: int) -> int:
    """Kernel nodes in the runner's two CUDA graphs (what one step launches)."""
    try:
        from cuda.bindings import runtime as rt
        n = 0
        for g in runner.graphs:
            err, nodes, cnt = rt.cudaGraphGetNodes(rt.cudaGraph_t(g.raw_cuda_graph()), 64)
            for nd in nodes[:cnt]:
                e, ty = rt.cudaGraphNodeGetType(nd)
                n += int(ty == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel)
        return n if n else fallback
    except Exception:
        return fallback


def sweep(fp, args, pk, flush, stream):
    """Per-length numbers at N = 1 (device-resident inputs, generated on the GPU from seed 5 with
    the same recipe): stage ms, density, effective TFLOP/s, attention fraction of burst bf16 peak,
    discovery fraction of HBM, speedup over the in-tree dense K5 and, as context only, cuDNN SDPA
    (torch) dense causal time."""
    import torch.nn.functional as F
    from paper_2603_06199_b200 import workload
    cfg = fp.PipelineConfig(alpha=args.alpha)
    tau = cfg.resolved_scale(D)
    res = []
    for L in SWEEP_LS:
        torch.cuda.empty_cache()
        q, k, v = workload.composite(5, 1, args.hq, args.hkv, L, device="cuda")
        M = (L + B - 1) // B
        r = fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16).capture()
        for _ in range(2):
            r.replay_discover()
            r.replay_attend()
        reps = 5 if L <= 32768 else 3
        ts = time_runner(r, stream, flush, reps)
        r.check()
        f_alg, visits, diag = plan_flops(r.counts, r.idx)
        ms_d, ms_a = statistics.median(ts["disc"]), statistics.median(ts["attn"])
        ms = ms_d + ms_a
        disc_bytes = args.hq * L * D * 2 + args.hkv * L * D * 2 + M * M * args.hq * 4 \
            + M * args.hq * 4
        t_dense = []
        for i in range(3):
            flush.fill_(2)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dres = fp.dense_attention(q, k, v, tau, out_dtype=torch.bfloat16)
            e1.record(stream)
            torch.cuda.synchronize()
            if i:
                t_dense.append(e0.elapsed_time(e1))
            del dres
        t_sdpa = None
        try:
            t_sdpa = []
            for i in range(3):
                flush.fill_(3)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True, scale=tau,
                                                   enable_gqa=True)
                e1.record(stream)
                torch.cuda.synchronize()
                if i:
                    t_sdpa.append(e0.elapsed_time(e1))
                del o
            t_sdpa = statistics.mean(t_sdpa)
        except Exception:
            t_sdpa = None
        ms_dense = statistics.mean(t_dense)
        fl = dense_flops(1, args.hq, L)
        tcfg = {"L": L, "hq": args.hq, "hkv": args.hkv, "alpha": args.alpha, "seed": 5,
                "gen": "cuda"}
        res.append({
            "L": L, "ms": ms, "discover_select_ms": ms_d, "sparse_attention_ms": ms_a,
            "eff_tflops": fl / (ms * 1e-3) / 1e12, "density": visits / (args.hq * M * (M + 1) / 2),
            "attn_alg_tflops": f_alg / (ms_a * 1e-3) / 1e12,
            "attn_frac_of_burst": f_alg / (ms_a * 1e-3) / 1e12 / pk["tc_burst"],
            "disc_gbps": disc_bytes / (ms_d * 1e-3) / 1e9,
            "disc_frac_of_hbm": disc_bytes / (ms_d * 1e-3) / 1e9 / pk["hbm"],
            "dense_k5_ms": ms_dense, "speedup_vs_dense_k5": ms_dense / ms,
            "sdpa_dense_ms": t_sdpa,
            "attn_traffic": ncu_traffic("fa_kernel", tcfg),
            "disc_traffic": ncu_traffic("discover_kernel", tcfg),
        })
        del r, q, k, v
    torch.cuda.empty_cache()
    return res


def run_gpu_arm(args, rank, world, dist):
    import paper_2603_06199_b200 as fp

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = fp.PipelineConfig(alpha=args.alpha)
    q_h, k_h, v_h = make_inputs(args)
    q, k, v = (x.to(dev) for x in (q_h, k_h, v_h))
    grid = fp.make_block_grid(args.L, B)
    M = grid.num_query_blocks
    tau = cfg.resolved_scale(D)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # this rank's share of the layer as two CUDA graph launches over preallocated buffers
    # (PrefillRunner): no host allocation, tensor-map encoding or synchronisation in the step
    runner, gather, (q_lo, q_hi) = make_runner(fp, args, q, k, v, cfg, world, rank)
    runner.capture()
    for _ in range(args.warmup):
        do_step(runner, gather)
    torch.cuda.synchronize()
    runner.check()  # PlanError surfaces here (plans come from discovery: never expected)

    with ClockSampler(dev.index) as clocks:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ts = time_runner(runner, stream, flush, args.steps, gather, dist)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    mine = [statistics.mean(ts[x]) for x in ("step", "disc", "attn", "gather")]
    per_rank = [mine]
    ms, ms_disc, ms_attn, ms_gather = mine
    rows = owned_rows(args, M, world, rank)
    f_alg, visits, diag = plan_totals(runner, rows)
    if dist:  # max over ranks; per-rank list; plan totals summed
        cd = _coll_device(dist, dev)
        allr = [torch.zeros(4, dtype=torch.float64, device=cd) for _ in range(world)]
        dist.all_gather(allr, torch.tensor(mine, dtype=torch.float64, device=cd))
        per_rank = [x.tolist() for x in allr]
        ms, ms_disc, ms_attn, ms_gather = (max(r[i] for r in per_rank) for i in range(4))
        tot = torch.tensor([visits, diag], dtype=torch.float64, device=cd)
        dist.all_reduce(tot)
        visits, diag = (int(x) for x in tot.tolist())
    dens = visits / (args.hq * M * (M + 1) / 2.0)
    f_alg_local = f_alg  # this rank's plan FLOPs (its kernel's roofline)

    # dense causal kernel (K5) in the same codebase: the speedup denominator (whole layer, 1 GPU)
    ms_dense = None
    if world == 1:
        t_dense = []
        for i in range(max(2, min(args.steps, 5)) + 1):
            flush.fill_(2)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fp.dense_attention(q, k, v, tau, out_dtype=torch.bfloat16)
            e1.record(stream)
            torch.cuda.synchronize()
            if i:
                t_dense.append(e0.elapsed_time(e1))
        ms_dense = statistics.mean(t_dense)

    # e2e through the reference-facing host-buffer C-ABI call (H2D + kernels + D2H each step);
    # at N > 1 each rank calls it on its KV-group shard (host outputs are not gathered)
    e2e_ms = None
    h2d = d2h = 0
    if not args.no_e2e:
        from paper_2603_06199_b200 import shard
        s = shard.kv_group_shard(args.hq, args.hkv, world, rank) if world > 1 else None
        src = shard.local_slices(q_h, k_h, v_h, s) if s else (q_h, k_h, v_h)
        qp, kp, vp = (x.contiguous().pin_memory() for x in src)
        outp = torch.empty(qp.shape, dtype=torch.bfloat16).pin_memory()
        lsep = torch.empty(qp.shape[:3], dtype=torch.float32).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in (qp, kp, vp))
        d2h = outp.numel() * 2 + lsep.numel() * 4
        fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
        times = []
        for _ in range(max(1, min(args.steps, 5))):
            flush.fill_(3)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
            times.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = statistics.mean(times)
        if dist:
            cd = _coll_device(dist, dev)
            tt = torch.tensor([e2e_ms, h2d, d2h], dtype=torch.float64, device=cd)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt[0])
            tt2 = torch.tensor([h2d, d2h], dtype=torch.float64, device=cd)
            dist.all_reduce(tt2)
            h2d, d2h = (int(x) for x in tt2.tolist())

    # CPU baseline + parity (rank 0, N = 1 only): the reference on this box's host cores on a
    # bounded sample of Q heads of the same layer; its plans and outputs are compared with the
    # GPU step's (oracle/parity.py bars)
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        heads = sample_heads(args.hq, args.hkv, args.cpu_heads or threads)
        qf, kf, vf = (x.float().numpy() for x in (q_h, k_h, v_h))
        r, kind = reference_pipeline(qf, kf, vf, args, threads, heads)
        cpu = {"value": dense_flops(1, len(heads), args.L) / r["secs"] / 1e12, "unit": UNIT,
               "cores": threads, "kind": kind,
               "sample": f"{len(heads)} of {args.hq} Q heads of this layer (L={args.L}), one per "
                         f"thread, {r['secs']:.1f} s; value normalised per head"}
        parity = compare_with_reference(runner, r, heads, args)

    if rank != 0:
        return
    pk = peaks()
    job_flops = dense_flops(1, args.hq, args.L)  # ONE layer, whatever N (strong scaling)
    value = job_flops / (ms * 1e-3) / 1e12
    achieved = f_alg_local / (ms_attn * 1e-3) / 1e12 if world == 1 else \
        f_alg_local / (statistics.mean(ts["attn"]) * 1e-3) / 1e12
    # discovery algorithmic bytes: read Q and K once, write idx (incl. fill) and counts
    disc_bytes = args.hq * args.L * D * 2 + args.hkv * args.L * D * 2 \
        + M * M * args.hq * 4 + M * args.hq * 4
    traffic_cfg = {"L": args.L, "hq": args.hq, "hkv": args.hkv, "alpha": args.alpha,
                   "seed": args.seed}
    launches = kernel_launches(runner, 3)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (vertical+slash composite planted in Q/K geometry, seeded)",
        "config": bench_config(args, world),
        "breakdown_ms": {"discover_select": ms_disc, "sparse_attention": ms_attn,
                         "gather": ms_gather, "dense_attention_k5": ms_dense},
        "density": dens, "block_visits": visits, "diag_visits": diag,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": pk["tc_burst"],
                     "unit": "TFLOP/s", "frac": achieved / pk["tc_burst"],
                     "peak_src": pk["src"] + " burst bf16 (cuBLAS 8192^3 at full clock; the step "
                                             "is a short burst at ~1965 MHz)",
                     "frac_of_sustained": achieved / pk["tc_sustained"],
                     "sustained_note": "sustained peak = cuBLAS back to back under the 1000 W "
                                       "power cap (1335 MHz median), not this step's regime",
                     "traffic": ncu_traffic("fa_kernel", traffic_cfg),
                     "traffic_unit": "DRAM bytes per step of this kernel (ncu --set full, cold L2; summed over its launches: one per KV-range phase)",
                     "kernel": "fa_kernel (K4, csrc/attention_fa.cu)"
                               + (" on rank 0's shard" if world > 1 else "")},
        "discovery_roofline": {"bound": "hbm", "kernel": "discover_kernel (pools K in-kernel) + select_rows",
                               "traffic": ncu_traffic("discover_kernel", traffic_cfg),
                               "achieved": disc_bytes / (ms_disc * 1e-3) / 1e9,
                               "peak": pk["hbm"], "unit": "GB/s",
                               "frac": disc_bytes / (ms_disc * 1e-3) / 1e9 / pk["hbm"],
                               "bytes": disc_bytes,
                               "tensor": discovery_tensor_view(args, M, ms_disc, pk)}
        if world == 1 else None,
        "clocks": clocks.summary(),
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
    }
    if ms_dense:
        out["speedup_vs_dense"] = ms_dense / ms
        out["speedup_attn_only"] = ms_dense / ms_attn
    if world > 1:
        out["per_rank_ms"] = [{"step": r[0], "discover_select": r[1], "sparse_attention": r[2],
                               "gather": r[3]} for r in per_rank]
        out["partition"] = args.partition
        if args.partition == "kv_zigzag" and getattr(args, "kv_weights_used", None):
            from paper_2603_06199_b200 import shard
            out["kv_group_ranks"] = shard.kv_group_ranks(args.hkv, world, args.kv_weights_used)
            out["kv_group_visits"] = args.kv_weights_used
    if e2e_ms is not None:
        out["e2e"] = {"value": job_flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT, "ms": e2e_ms,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "path": "fpb_host_prefill (pinned host buffers)"
                              + (", per rank on its KV-group shard" if world > 1 else "")}
    if cpu:
        out["cpu_baseline"] = cpu
    if parity:
        out["parity"] = parity
    if world == 1 and not args.no_sweep:
        out["sweep"] = sweep(fp, args, pk, flush, stream)
    print(json.dumps(out), flush=True)


def compare_with_reference(runner, r, heads, args):
    """The GPU step's plan and (bf16) output on the sampled heads against the reference's."""
    import numpy as np
    from oracle import parity as P
    if "idx" not in r:
        return None
    g_idx = np.stack([runner.idx[0, :, :, h].cpu().numpy() for h in heads])
    g_cnt = np.stack([runner.counts[0, :, h].cpu().numpy() for h in heads])
    pp = P.compare_plans(g_idx, g_cnt, r["idx"], r["counts"], r["score"], args.alpha)
    g_out = np.stack([runner.out[0, h].float().cpu().numpy() for h in heads])
    g_lse = np.stack([runner.lse[0, h].cpu().numpy() for h in heads])
    po = P.compare_outputs(g_out, g_lse, r["out"], r["lse"], pp["same_row"], B)
    res = {k: v for k, v in pp.items() if k != "same_row"}
    res.update(po)
    res.update({"heads": len(heads), "mask_eps": P.MASK_EPS,
                "bars": "mask/idx/counts bit-exact outside the eps band; out & lse max-abs <= "
                        "2e-2, mean-abs <= 1e-3 (bf16 out vs reference fp32)",
                "ok": P.within_bars(po, pp)})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fpb200", choices=["fpb200", "reference"])
    ap.add_argument("--partition", default="kv", choices=["kv", "kv_zigzag", "rows", "zigzag"])
    ap.add_argument("--kv-weights", default="plan", choices=["plan", "equal"],
                    help="kv_zigzag: ranks per KV group by the calibration plan's visits per "
                         "group (plan) or world / Hkv each (equal)")
    ap.add_argument("--gather-chunks", type=int, default=2,
                    help="kv partition, N > 1: compute a rank's Q heads in this many chunks and "
                         "send each chunk's O/LSE while the next computes (1 = one all-gather "
                         "after all kernels)")
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=0.12)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--n-vertical", type=int, default=8)
    ap.add_argument("--n-slash", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-heads", type=int, default=0)
    ap.add_argument("--ref-heads", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1 and args.impl == "fpb200":
        import torch.distributed as tdist
        if os.environ.get("FPB_BENCH_SHARED_GPU"):
            # test mode for 1-GPU boxes: every rank on cuda:0, collectives over gloo
            os.environ["LOCAL_RANK"] = "0"
            tdist.init_process_group("gloo")
        else:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            tdist.init_process_group("nccl", device_id=torch.device(
                "cuda", int(os.environ.get("LOCAL_RANK", 0))))
        dist = tdist
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_gpu_arm(args, rank, world, dist)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
