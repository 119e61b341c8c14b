"""Build libfpb200.so in-tree: nvcc for sm_100a, explicit -gencode (no torch arch list)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["abi.cu", "pool.cu", "select.cu", "discover.cu", "attention.cu", "attention_fa.cu",
           "generic.cu", "baselines.cu"]
HEADERS = ["fp_ptx.cuh", "fp_common.cuh", "fp_kernels.h"]
LIB = os.path.join(HERE, "libfpb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "fpb200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if not force and out == LIB and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out + ".tmp",
           *[os.path.join(CSRC, f) for f in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    os.replace(out + ".tmp", out)
    if out == LIB:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
            f.write(res.stderr)
    if verbose:
        print(res.stderr)
    return out


ROOT = os.path.dirname(HERE)
CLI = os.path.join(HERE, "fpb200_cli")
CLI_SOURCES = [os.path.join(ROOT, "tools", "fpb200_cli.cpp"),
               os.path.join(ROOT, "tools", "cli", "json.hpp"),
               os.path.join(ROOT, "tools", "cli", "workloads.hpp"),
               os.path.join(ROOT, "include", "fpb200", "bsattn.hpp"),
               os.path.join(ROOT, "include", "fpb200", "fpt1.hpp"),
               os.path.join(ROOT, "include", "fpb200.h")]


def build_cli(force: bool = False) -> str:
    """The reference-compatible CLI (tools/fpb200_cli.cpp) linked against libfpb200.so ($ORIGIN rpath)."""
    build()
    if (not force and os.path.exists(CLI)
            and all(os.path.getmtime(p) <= os.path.getmtime(CLI) for p in CLI_SOURCES + [LIB])):
        return CLI
    cmd = [os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-Wall", "-Wextra",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "tools"),
           CLI_SOURCES[0], f"-L{HERE}", "-l:libfpb200.so", "-Wl,-rpath,$ORIGIN", "-o", CLI + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("g++ failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    os.replace(CLI + ".tmp", CLI)
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
    print(build_cli(force="--force" in sys.argv))
