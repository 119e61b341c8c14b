"""CPU-only tests: the C-ABI library loads and exports every declared symbol; host-side logic
(grid, config validation, sharding, workload, error behaviour) mirrors the reference; the product
path refuses CPU tensors (no fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_06199_b200 import build
    build.build()
    from paper_2603_06199_b200 import _abi
    return _abi.lib()


def test_abi_exports_every_header_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "fpb200.h")).read()
    declared = sorted(set(re.findall(r"\b(fpb_\w+)\s*\(", hdr)))
    from paper_2603_06199_b200 import _abi
    assert declared == sorted(_abi.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_validation_without_gpu(lib):
    """Pure host-side validation paths of the ABI (no device work is issued)."""
    from paper_2603_06199_b200 import _abi
    p = _abi.Problem()
    lib.fpb_problem_init(ctypes.byref(p), 1, 32, 4, 32768, 128)
    assert (p.block_size, p.sink_tokens, p.window_tokens) == (128, 256, 512)
    assert abs(p.alpha - 0.12) < 1e-7 and p.scale == 0.0
    n = ctypes.c_size_t(0)
    assert lib.fpb_workspace_bytes(ctypes.byref(p), _abi.FPB_BF16, ctypes.byref(n)) == 0
    assert n.value >= 1024 + 2 * 4 * 256 * 128 * 2  # >= scheduler counter + k̄ hi/lo split
    bad = _abi.Problem()
    lib.fpb_problem_init(ctypes.byref(bad), 1, 6, 4, 100, 128)  # Hq % Hkv != 0
    assert lib.fpb_workspace_bytes(ctypes.byref(bad), 1, ctypes.byref(n)) == _abi.FPB_EVALIDATION
    assert b"multiple" in lib.fpb_last_error()
    lib.fpb_problem_init(ctypes.byref(bad), 1, 4, 4, 100, 128)
    bad.alpha = -1.0  # ConfigError (core.hpp:98)
    assert lib.fpb_workspace_bytes(ctypes.byref(bad), 1, ctypes.byref(n)) == _abi.FPB_EVALIDATION
    bad.alpha, bad.window_tokens = 0.1, 0  # core.hpp:99
    assert lib.fpb_workspace_bytes(ctypes.byref(bad), 1, ctypes.byref(n)) == _abi.FPB_EVALIDATION
    bad.window_tokens, bad.d = 512, 64  # other head dims run the generic SIMT kernels
    assert lib.fpb_workspace_bytes(ctypes.byref(bad), 1, ctypes.byref(n)) == 0
    bad.d = 4096  # beyond the supported range
    assert lib.fpb_workspace_bytes(ctypes.byref(bad), 1, ctypes.byref(n)) == _abi.FPB_EVALIDATION
    assert lib.fpb_pool_keys(ctypes.byref(p), 1, None, None, None) == _abi.FPB_EUSAGE


def test_grid_and_config_mirror_reference():
    import paper_2603_06199_b200 as fp
    g = fp.make_block_grid(1000, 128)  # core.hpp:31-41
    assert (g.num_query_blocks, g.last_block_len, g.block_len(7), g.block_len(0)) == (8, 104, 104, 128)
    with pytest.raises(fp.ValidationError):
        fp.make_block_grid(0, 128)
    c = fp.PipelineConfig()
    assert c.sink_blocks() == 2 and c.window_blocks() == 4  # test_core.cpp:170-187
    assert abs(c.resolved_scale(128) - 1 / np.sqrt(128)) < 1e-7
    with pytest.raises(fp.ConfigError):
        fp.PipelineConfig(alpha=-0.1).validate()
    with pytest.raises(fp.ConfigError):
        fp.PipelineConfig(window_tokens=0).validate()
    with pytest.raises(fp.ConfigError):
        fp.PipelineConfig(epsilon=0).validate()
    assert issubclass(fp.PlanError, fp.ValidationError) and issubclass(fp.ConfigError, fp.ValidationError)


def test_product_refuses_cpu_tensors():
    """No CPU fallback: host tensors are rejected before any compute."""
    import paper_2603_06199_b200 as fp
    q = torch.zeros(1, 2, 256, 128, dtype=torch.bfloat16)
    with pytest.raises(fp.ValidationError):
        fp.discover(q, q, fp.make_block_grid(256, 128), 0.088)
    with pytest.raises(fp.ValidationError):
        fp.dense_attention(q, q, q, 0.088)


def test_kv_group_shard():
    from paper_2603_06199_b200.shard import kv_group_shard, unit_shard
    # Llama-3.1-8B: 32 Q / 8 KV at 1/2/4/8 GPUs
    for G in (1, 2, 4, 8):
        sh = [kv_group_shard(32, 8, G, r) for r in range(G)]
        assert [s.hq for s in sh] == [32 // G] * G and [s.hkv for s in sh] == [8 // G] * G
        assert sh[0].q_lo == 0 and sh[-1].q_hi == 32
        for s in sh:
            assert s.q_lo // 4 == s.kv_lo and (s.q_hi - 1) // 4 == s.kv_hi - 1
    # Qwen3: 32 Q / 4 KV on 8 GPUs -> 4 Q heads per rank, KV head replicated across 2 ranks
    sh = [kv_group_shard(32, 4, 8, r) for r in range(8)]
    assert [(s.q_lo, s.kv_lo) for s in sh] == [(0, 0), (4, 0), (8, 1), (12, 1), (16, 2), (20, 2),
                                              (24, 3), (28, 3)]
    with pytest.raises(ValueError):
        kv_group_shard(32, 4, 3, 0)
    assert [len(unit_shard(10, 4, r)) for r in range(4)] == [3, 3, 2, 2]


def test_workload_deterministic_and_shaped():
    from paper_2603_06199_b200 import workload
    a = workload.composite(5, 1, 4, 2, 512, n_vertical=2, n_slash=1)
    b = workload.composite(5, 1, 4, 2, 512, n_vertical=2, n_slash=1)
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    assert a[0].shape == (1, 4, 512, 128) and a[1].shape == (1, 2, 512, 128)
    assert a[0].dtype == torch.bfloat16


def test_bench_helpers():
    import bench
    counts = torch.tensor([[[1], [2]]], dtype=torch.int32)  # Z=1, M=2, H=1
    idx = torch.tensor([[[[0], [2]], [[0], [1]]]], dtype=torch.int32)
    f, visits, diag = bench.plan_flops(counts, idx)
    assert visits == 3 and diag == 2
    assert f == 4 * 128 * (1 * 128 * 128 + 2 * 128 * 129 / 2)
    assert bench.sample_heads(32, 4, 4) == [0, 8, 16, 24]
    assert bench.dense_flops(1, 32, 32768) == pytest.approx(8.796e12, rel=1e-3)
