#!/usr/bin/env python
"""FlashPrefill B200 benchmark — sparse-prefill attention on the Qwen3-30B-A3B layer shape.

One step = the whole FlashPrefill hot path over one synthetic batch resident in HBM:
  fpb_discover_select (K1 pooling + K2/K3 fused tcgen05 discovery, threshold, compaction)
  -> fpb_block_sparse_attention (K4 tcgen05 block-sparse FlashAttention).
Metric: effective TFLOP/s = dense-causal-equivalent FLOPs 4*d*Z*Hq*L(L+1)/2 / step time
(SURVEY §8d), whole job over all ranks; ms_per_step is reported beside it.

  python bench.py [--gpus N --steps K --warmup W] [--impl fpb200|reference] [--L 32768]
  N > 1: torchrun, one rank per GPU, weak scaling: rank r owns work units (sequence r, all KV-head
  groups) — the path shards by (sequence, KV-head group) with no data-path collective.

L2 hygiene: a 512 MiB buffer is written between timed steps (L2 is 126 MB); each step is timed
with CUDA events on the launching stream; max over ranks.
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
    committed `ncu --set full` capture (profiles/ncu_traffic.json, written by
    tools/ncu_summary.py --traffic); None unless the capture was taken on this exact config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f)[kernel]
    except (OSError, KeyError, ValueError):
        return None
    if any(rec.get("config", {}).get(k) != v for k, v in cfg.items()):
        return None
    return rec["dram_bytes"]


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


def plan_flops(counts: torch.Tensor, idx: torch.Tensor):
    """Algorithmic FLOPs of the visited blocks: 4 d B^2 off-diagonal, 4 d B(B+1)/2
    on the diagonal, plus the visit split."""
    Z, M, H = counts.shape
    c = counts.to(torch.int64)
    visits = int(c.sum())
    # diagonal visited iff block i appears in row (z, i, :, h) within the first C slots
    ar = torch.arange(M, device=idx.device)
    slot = torch.arange(M, device=idx.device).view(1, 1, M, 1)
    within = slot < counts.view(Z, M, 1, H)
    diag = int(((idx == ar.view(1, M, 1, 1)) & within).sum())
    f = 4.0 * D * ((visits - diag) * B * B + diag * B * (B + 1) / 2.0)
    return f, visits, diag


def make_inputs(args, seq_index: int):
    from paper_2603_06199_b200 import workload
    return workload.composite(args.seed + seq_index, 1, args.hq, args.hkv, args.L,
                              n_vertical=args.n_vertical, n_slash=args.n_slash)


# ------------------------------------------------------------------------------ CPU reference
def cpu_reference_step(q, k, v, args, threads: int, heads: list[int]):
    """Reference pipeline (oracle/_ref = the unmodified reference headers; port if absent) on the
    given (z*Hq + h) slices.  Returns (seconds, kind, visits)."""
    from oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    tau = float(1.0 / math.sqrt(D))
    secs, _, _, visits = o.pipeline(q, k, v, B, args.alpha, 256, 512, tau, 1e-10, heads, threads)
    return secs, kind, visits


def sample_heads(Hq: int, Hkv: int, n: int) -> list[int]:
    """Spread the sample over KV groups: head order 0, g, 2g, ..., 1, g+1, ..."""
    g = Hq // Hkv
    order = [kh * g + j for j in range(g) for kh in range(Hkv)]
    return order[:max(1, min(n, Hq))]


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    q, k, v = make_inputs(args, 0)
    qf, kf, vf = (x.float().numpy() for x in (q, k, v))
    heads = sample_heads(args.hq, args.hkv, args.ref_heads or threads)
    times = []
    kind = None
    for i in range(args.warmup + args.steps):
        secs, kind, visits = cpu_reference_step(qf, kf, vf, args, threads, heads)
        if i >= args.warmup:
            times.append(secs)
    t = statistics.mean(times)
    flops = dense_flops(1, len(heads), args.L)
    value = flops / t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (vertical+slash composite, seeded; bf16 values upcast exactly)",
        "config": {"workload": f"Qwen3-30B-A3B layer (Hq={args.hq}, Hkv={args.hkv}, d=128) "
                               f"bf16 causal L={args.L}, alpha={args.alpha}",
                   "sample_heads": len(heads), "L": args.L},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{len(heads)} of {args.hq} Q heads per step, full L={args.L}, "
                                   f"discover->mask->compress->sparse attention per head"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def _coll_device(dist, dev):
    return torch.device("cpu") if dist.get_backend() == "gloo" else dev


def run_gpu_arm(args, rank, world, dist):
    import paper_2603_06199_b200 as fp

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = fp.PipelineConfig(alpha=args.alpha)
    q_h, k_h, v_h = make_inputs(args, rank)
    q, k, v = (x.to(dev) for x in (q_h, k_h, v_h))
    grid = fp.make_block_grid(args.L, B)
    tau = cfg.resolved_scale(D)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # the step as two CUDA graph launches over preallocated buffers (PrefillRunner): no host
    # allocation, tensor-map encoding or synchronisation inside the timed region
    runner = fp.PrefillRunner(q, k, v, cfg, out_dtype=torch.bfloat16)
    if not args.no_graphs:
        runner.capture()

    def step():
        runner.replay_discover()
        e_mid.record(stream)
        runner.replay_attend()
        return runner.plan, runner

    e_mid = torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        plan, res = step()
    torch.cuda.synchronize()
    runner.check()  # PlanError surfaces here (plans come from discovery: never expected)

    t_step, t_disc, t_attn = [], [], []
    with ClockSampler(dev.index) as clocks:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1)  # evict L2 between steps (not timed)
            e0, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_mid = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plan, res = step()
            e2.record(stream)
            torch.cuda.synchronize()
            t_step.append(e0.elapsed_time(e2))
            t_disc.append(e0.elapsed_time(e_mid))
            t_attn.append(e_mid.elapsed_time(e2))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms = statistics.mean(t_step)
    ms_disc, ms_attn = statistics.mean(t_disc), statistics.mean(t_attn)
    if dist:  # max over ranks
        tt = torch.tensor([ms, ms_disc, ms_attn], device=_coll_device(dist, dev))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, ms_disc, ms_attn = (float(x) for x in tt.tolist())

    f_alg, visits, diag = plan_flops(plan.counts, plan.indices)
    M = grid.num_query_blocks
    dens = visits / (args.hq * M * (M + 1) / 2.0)

    # dense causal kernel (K5) in the same codebase: the speedup denominator
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

    # e2e through the reference-facing host-buffer C-ABI call (H2D + kernels + D2H each step)
    e2e_ms = None
    h2d = d2h = 0
    if not args.no_e2e:
        qp, kp, vp = (x.pin_memory() for x in (q_h, k_h, v_h))
        outp = torch.empty(qp.shape, dtype=torch.bfloat16).pin_memory()
        lsep = torch.empty(qp.shape[:3], dtype=torch.float32).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in (qp, kp, vp))
        d2h = outp.numel() * 2 + lsep.numel() * 4
        for _ in range(1):
            fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
        times = []
        for _ in range(max(1, min(args.steps, 5))):
            flush.fill_(3)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fp.prefill_host(qp, kp, vp, cfg, outp, lsep)
            times.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = statistics.mean(times)
        if dist:
            tt = torch.tensor([e2e_ms], device=_coll_device(dist, dev))
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())

    # CPU baseline (rank 0, N = 1 only): reference on this box's host cores, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        heads = sample_heads(args.hq, args.hkv, args.cpu_heads or threads)
        qf, kf, vf = (x.float().numpy() for x in (q_h, k_h, v_h))
        secs, kind, _ = cpu_reference_step(qf, kf, vf, args, threads, heads)
        cpu = {"value": dense_flops(1, len(heads), args.L) / secs / 1e12, "unit": UNIT,
               "cores": threads, "kind": kind,
               "sample": f"{len(heads)} of {args.hq} Q heads of this workload (L={args.L}), "
                         f"one per thread, {secs:.1f} s"}

    if rank != 0:
        return
    pk = peaks()
    job_flops = dense_flops(world, args.hq, args.L)  # world sequences (weak scaling)
    value = job_flops / (ms * 1e-3) / 1e12
    achieved = f_alg / (ms_attn * 1e-3) / 1e12  # per GPU, attention kernel (dominant)
    # discovery algorithmic bytes: read Q and K once, write idx (incl. fill) and counts
    disc_bytes = args.hq * args.L * D * 2 + args.hkv * args.L * D * 2 \
        + M * M * args.hq * 4 + M * args.hq * 4
    traffic_cfg = {"L": args.L, "hq": args.hq, "hkv": args.hkv, "alpha": args.alpha,
                   "seed": args.seed}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (vertical+slash composite planted in Q/K geometry, seeded)",
        "config": {"workload": f"Qwen3-30B-A3B attention layer (Hq={args.hq}, Hkv={args.hkv}, "
                               f"d=128) bf16 causal L={args.L} per GPU, alpha={args.alpha}, "
                               f"B=128, sink 256, window 512",
                   "global_batch_sequences": world, "seq_len": args.L,
                   "parallelism": f"shard (sequence, KV-head group) units over {world} GPU(s), "
                                  f"no data-path collective",
                   "l2": "512 MiB buffer written between timed steps (L2 126 MB)",
                   "launch": "CUDA graphs (PrefillRunner.capture)" if not args.no_graphs
                             else "direct C-ABI launches"},
        "breakdown_ms": {"discover_select": ms_disc, "sparse_attention": ms_attn,
                         "dense_attention_k5": ms_dense},
        "speedup_vs_dense": ms_dense / ms, "speedup_attn_only": ms_dense / ms_attn,
        "density": dens, "block_visits": visits, "diag_visits": diag,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": pk["tc_sustained"],
                     "unit": "TFLOP/s", "frac": achieved / pk["tc_sustained"],
                     "frac_of_burst": achieved / pk["tc_burst"],
                     "traffic": ncu_traffic("fa_kernel", traffic_cfg),
                     "traffic_unit": "bytes per launch (ncu --set full, cold L2)",
                     "kernel": "fa_kernel (K4, csrc/attention_fa.cu)", "peak_src": pk["src"] + " sustained"},
        "discovery_roofline": {"bound": "hbm", "kernel": "discover_kernel (K2+K3)",
                               "traffic": ncu_traffic("discover_kernel", traffic_cfg), "achieved": disc_bytes / (ms_disc * 1e-3) / 1e9,
                               "peak": pk["hbm"], "unit": "GB/s",
                               "frac": disc_bytes / (ms_disc * 1e-3) / 1e9 / pk["hbm"],
                               "bytes": disc_bytes},
        "clocks": clocks.summary(),
        "gpu_launches": 3 * args.steps,
    }
    if e2e_ms is not None:
        out["e2e"] = {"value": job_flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT, "ms": e2e_ms,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    if cpu:
        out["cpu_baseline"] = cpu
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fpb200", choices=["fpb200", "reference"])
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=0.12)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--n-vertical", type=int, default=8)
    ap.add_argument("--n-slash", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true",
                    help="launch the two stages directly instead of replaying CUDA graphs")
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
            # test mode for 1-GPU boxes: every rank on cuda:0, timing collectives over gloo
            os.environ["LOCAL_RANK"] = "0"
            tdist.init_process_group("gloo")
        else:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            tdist.init_process_group("nccl")
        dist = tdist
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_gpu_arm(args, rank, world, dist)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
