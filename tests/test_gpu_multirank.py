"""The N > 1 path with the REAL kernels: several ranks share cuda:0 (the pool gives one GPU per
box) and talk over gloo; each rank runs its shard of one layer through PrefillRunner (the bench's
CUDA-graph step) and the gather reassembles O and LSE.  The gathered result must be bit-identical
to the unsharded call — every (z, h, query block) is computed independently (discovery.hpp:87-88,
selection.hpp:71-72, attention.hpp:59-60), so sharding may not change a single bit.

Also runs bench.py itself under torchrun in that shared-GPU mode (FPB_BENCH_SHARED_GPU=1) and
checks its strong-scaling line."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, part, shape, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import paper_2603_06199_b200 as fp
    from paper_2603_06199_b200 import shard
    torch.cuda.set_device(0)
    Hq, Hkv, L = shape
    q, k, v = (x.cuda() for x in fp.workload.composite(17, 1, Hq, Hkv, L))
    cfg = fp.PipelineConfig(alpha=0.12)
    if part == "kv":
        s = shard.kv_group_shard(Hq, Hkv, world, rank)
        r = fp.PrefillRunner(*shard.local_slices(q, k, v, s), cfg).capture()
        r.replay_discover()
        r.replay_attend()
        out, lse = shard.gather_heads(r.out, r.lse, Hq, Hkv)
    elif part == "kv_chunked":  # bench.py's overlapped gather: head chunks, P2P per chunk
        s = shard.kv_group_shard(Hq, Hkv, world, rank)
        ql, kl, vl = shard.local_slices(q, k, v, s)
        out = torch.empty(q.shape, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
        g = shard.OverlappedHeadGather(Hq, Hkv, out, lse)
        rs = []
        for a, b in shard.head_chunks(s.hq, 2):
            r = fp.PrefillRunner(ql[:, a:b].contiguous(), kl, vl, cfg).capture()
            r.replay_discover()
            r.replay_attend()
            g.post(a, b, r.out, r.lse)
            rs.append(r)
        g.wait()
        r = rs[0]
    elif part.startswith("api_"):  # the one-call API: shard.prefill_sharded
        out, lse = shard.prefill_sharded(q, k, v, cfg, partition=part[4:])
        r = None
    elif part in ("kv_zigzag", "kv_weighted"):
        # one KV head per rank, a group's ranks split by zigzag rows; kv_weighted: ranks per group
        # by the layer plan's visits per group (3 ranks over 2 groups: 2 + 1)
        w = None
        if part == "kv_weighted":
            cnt = fp.discover_select(q, k, cfg)[0].counts.sum(dim=(0, 1)).double()
            g = Hq // Hkv
            w = [float(cnt[i * g:(i + 1) * g].sum()) for i in range(Hkv)]
        s, rows = shard.kv_zigzag_shard(Hq, Hkv, world, rank, w)
        r = fp.PrefillRunner(*shard.local_slices(q, k, v, s), cfg, rows=rows).capture()
        r.replay_discover()
        r.replay_attend()
        out, lse = shard.gather_kv_zigzag(r.out, r.lse, Hq, Hkv, 128, weights=w)
    else:
        rows = shard.row_shard(world, rank) if part == "rows" else shard.zigzag_shard(world, rank)
        r = fp.PrefillRunner(q, k, v, cfg, rows=rows).capture()
        r.replay_discover()
        r.replay_attend()
        g = shard.gather_rows if part == "rows" else shard.gather_zigzag
        out, lse = g(r.out, r.lse, 128)
    if r is not None:
        r.check()
    if rank == 0:
        ret["out"] = out.cpu()
        ret["lse"] = lse.cpu()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("part,world,shape", [
    ("kv", 2, (8, 2, 2048)),     # one KV group per rank
    ("kv", 4, (8, 2, 2048)),     # world > Hkv: each group's 4 Q heads split 2 + 2
    ("kv_chunked", 2, (8, 2, 2048)),  # 4 Q heads per rank in 2 chunks, P2P gather per chunk
    ("kv_chunked", 4, (12, 2, 1000)),  # 3 Q heads per rank: chunks of 2 + 1, ragged L
    ("rows", 2, (8, 2, 3000)),   # interleaved query blocks, ragged last block
    ("zigzag", 3, (8, 2, 3000)),
    ("kv_zigzag", 4, (8, 2, 3000)),  # 2 ranks per KV group, each with the group's 4 Q heads
    ("kv_weighted", 3, (8, 2, 3000)),  # ranks per KV group by plan visits (2 + 1)
    ("api_kv", 2, (8, 2, 2048)),       # shard.prefill_sharded, each partition
    ("api_kv_zigzag", 4, (8, 2, 2500)),
    ("api_zigzag", 3, (4, 2, 1700)),
])
def test_sharded_layer_gathers_bit_identical(fp, part, world, shape):
    Hq, Hkv, L = shape
    q, k, v = (x.cuda() for x in fp.workload.composite(17, 1, Hq, Hkv, L))
    r = fp.PrefillRunner(q, k, v, fp.PipelineConfig(alpha=0.12))
    r.discover()
    r.attend()
    torch.cuda.synchronize()
    mgr = mp.get_context("spawn").Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), part, shape, ret), nprocs=world, join=True)
    assert torch.equal(ret["out"], r.out.cpu()), part
    assert torch.equal(ret["lse"], r.lse.cpu()), part


@pytest.mark.parametrize("part,chunks,extra", [("kv", 2, []), ("kv", 1, []), ("rows", 1, []),
                                               ("kv_zigzag", 1, ["--hq", "16", "--hkv", "1"])])
def test_bench_two_ranks_shared_gpu(fp, part, chunks, extra):
    """bench.py --gpus 2 under torchrun (shared-GPU gloo mode): one strong-scaling JSON line with
    per-rank times and the gather inside the step (kv: chunked P2P gather overlapped with the
    next chunk's compute, or one all-gather after all kernels)."""
    env = dict(os.environ, FPB_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--L", "8192", "--no-e2e",
           "--partition", part, "--gather-chunks", str(chunks)] + extra
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [x for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, res.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong" and rec["partition"] == part
    assert len(rec["per_rank_ms"]) == 2
    assert rec["ms_per_step"] >= max(x["step"] for x in rec["per_rank_ms"]) - 1e-9
    assert rec["breakdown_ms"]["gather"] > 0
    assert 0 < rec["density"] <= 1 and rec["gpu_launches"] >= 3 * rec["steps"]
