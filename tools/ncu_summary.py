#!/usr/bin/env python
"""Summarise an ncu --set full report (raw page) into the metrics the roofline argument needs.

usage: python tools/ncu_summary.py gpurun_out/r1_attn.ncu-rep [more.ncu-rep ...]
       python tools/ncu_summary.py --traffic KERNEL 'CONFIG_JSON' rep.ncu-rep
           records that kernel's per-launch DRAM bytes (read + write) in profiles/ncu_traffic.json
           (one record per config), which bench.py reports as roofline.traffic / the sweep's
           attn_traffic / disc_traffic when its config matches CONFIG_JSON.
"""
import json
import os
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active (realtime) %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"{path}: no data\n"
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"kernel: {name[:120]}")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {label:34s} {r[i]:>16s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(r[i]), h.split("stalled_")[1].replace(".ratio", "")))
                except ValueError:
                    pass
            elif h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i]), "pc:" + h.split("stalled_")[1]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            out.append("  top stall reasons: " + ", ".join(f"{n}={v:.3g}" for v, n in stalls[:8]))
    return "\n".join(out) + "\n"


_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(path, kernel, cfg):
    """DRAM bytes (read + write) of one step's launches of `kernel` in the report, summed (the
    attention kernel runs one launch per KV-range phase), filed under `cfg`."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    tot, n = 0.0, 0
    for r in rows[2:]:
        if kernel not in r[hdr.index("Kernel Name")]:
            continue
        n += 1
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(key)
            tot += float(r[i].replace(",", "")) * _SCALE[units[i]]
    if not n:
        raise SystemExit(f"{kernel} not in {path}")
    dest = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "ncu_traffic.json")
    data = json.load(open(dest)) if os.path.exists(dest) else {}
    recs = data.get(kernel, [])
    recs = recs if isinstance(recs, list) else [recs]
    recs = [x for x in recs if x.get("config") != cfg]  # one record per config
    recs.append({"dram_bytes": tot, "launches": n, "config": cfg,
                 "capture": os.path.basename(path)})
    data[kernel] = recs
    with open(dest, "w") as f:
        json.dump(data, f, indent=1)
    return tot


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        print(traffic(sys.argv[4], sys.argv[2], json.loads(sys.argv[3])))
        sys.exit(0)
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summarise(p))
