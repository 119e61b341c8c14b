"""ctypes binding of libfpb200.so (include/fpb200.h).  No torch types cross the boundary.

Loading fails loudly when the library is missing: there is no CPU fallback anywhere in the
product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPB200_LIB") or os.path.join(HERE, "libfpb200.so")

FPB_OK, FPB_EUSAGE, FPB_EVALIDATION, FPB_EFORMAT, FPB_ECUDA = 0, 1, 2, 3, 4
FPB_F32, FPB_BF16 = 0, 1

# Every symbol include/fpb200.h declares (checked by tests/test_abi_symbols.py).
EXPORTS = [
    "fpb_problem_init", "fpb_version", "fpb_last_error", "fpb_workspace_bytes",
    "fpb_pool_keys", "fpb_approx_block_scores", "fpb_normalize_block_scores", "fpb_discover",
    "fpb_max_threshold_mask", "fpb_compress_indices", "fpb_discover_select", "fpb_visit_count",
    "fpb_block_sparse_attention", "fpb_dense_attention", "fpb_full_causal_plan",
    "fpb_discover_select_rows", "fpb_block_sparse_attention_rows",
    "fpb_discover_select_zigzag", "fpb_block_sparse_attention_zigzag",
    "fpb_topk_select", "fpb_topp_select", "fpb_baseline_workspace_bytes",
    "fpb_discover_pool_both", "fpb_discover_exact",
    "fpb_host_pool_keys", "fpb_host_approx_block_scores", "fpb_host_normalize_block_scores",
    "fpb_host_discover", "fpb_host_max_threshold_mask", "fpb_host_compress_indices",
    "fpb_host_topk_select", "fpb_host_topp_select", "fpb_host_discover_method",
    "fpb_host_block_sparse_attention", "fpb_host_dense_attention", "fpb_host_prefill",
]


class Problem(C.Structure):
    """fpb_problem (include/fpb200.h) == shapes + PipelineConfig (core.hpp:87-112)."""

    _fields_ = [
        ("Z", C.c_int64), ("Hq", C.c_int64), ("Hkv", C.c_int64), ("L", C.c_int64),
        ("d", C.c_int64), ("block_size", C.c_int32), ("alpha", C.c_float),
        ("sink_tokens", C.c_int32), ("window_tokens", C.c_int32), ("scale", C.c_float),
        ("epsilon", C.c_float),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load libfpb200.so (never a fallback: raises if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2603_06199_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER(Problem)
        p, u64p = C.c_void_p, C.POINTER(C.c_uint64)
        sig = {
            "fpb_problem_init": (None, [P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
            "fpb_version": (C.c_int, []),
            "fpb_last_error": (C.c_char_p, []),
            "fpb_workspace_bytes": (C.c_int, [P, C.c_int, C.POINTER(C.c_size_t)]),
            "fpb_pool_keys": (C.c_int, [P, C.c_int, p, p, p]),
            "fpb_approx_block_scores": (C.c_int, [P, C.c_int, p, p, p, p, p, C.c_size_t, p]),
            "fpb_normalize_block_scores": (C.c_int, [P, p, p, p, p]),
            "fpb_discover": (C.c_int, [P, C.c_int, p, p, p, p, p, p, C.c_size_t, p]),
            "fpb_max_threshold_mask": (C.c_int, [P, p, p, p, p]),
            "fpb_compress_indices": (C.c_int, [P, p, p, p, p]),
            "fpb_discover_select": (C.c_int, [P, C.c_int, p, p, p, p, p, p, p, p, p, C.c_size_t,
                                              p]),
            "fpb_discover_select_rows": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int, p, p, p,
                                                   p, p, p, p, p, p, C.c_size_t, p]),
            "fpb_block_sparse_attention_rows": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int, p, p,
                                                          p, p, p, C.c_int, p, p, p, p, p,
                                                          C.c_size_t, p]),
            "fpb_discover_select_zigzag": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int, p, p, p,
                                                     p, p, p, p, p, p, C.c_size_t, p]),
            "fpb_block_sparse_attention_zigzag": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int, p,
                                                            p, p, p, p, C.c_int, p, p, p, p, p,
                                                            C.c_size_t, p]),
            "fpb_visit_count": (C.c_int, [P, p, p, p]),
            "fpb_block_sparse_attention": (C.c_int, [P, C.c_int, p, p, p, p, p, C.c_int, p, p, p,
                                                     p, p, C.c_size_t, p]),
            "fpb_dense_attention": (C.c_int, [P, C.c_int, p, p, p, C.c_int, p, p, p, C.c_size_t,
                                              p]),
            "fpb_full_causal_plan": (C.c_int, [P, p, p, p]),
            "fpb_topk_select": (C.c_int, [P, p, C.c_int32, p, p]),
            "fpb_topp_select": (C.c_int, [P, p, C.c_float, p, p]),
            "fpb_baseline_workspace_bytes": (C.c_int, [P, C.POINTER(C.c_size_t)]),
            "fpb_discover_pool_both": (C.c_int, [P, C.c_int, p, p, p, p, p, p, C.c_size_t, p]),
            "fpb_discover_exact": (C.c_int, [P, C.c_int, p, p, p, p, p, p, C.c_size_t, p]),
            "fpb_host_topk_select": (C.c_int, [P, p, C.c_int32, p]),
            "fpb_host_topp_select": (C.c_int, [P, p, C.c_float, p]),
            "fpb_host_discover_method": (C.c_int, [P, C.c_int, C.c_int, p, p, p, p, p]),
            "fpb_host_pool_keys": (C.c_int, [P, C.c_int, p, p]),
            "fpb_host_approx_block_scores": (C.c_int, [P, C.c_int, p, p, p, p]),
            "fpb_host_normalize_block_scores": (C.c_int, [P, p, p, p]),
            "fpb_host_discover": (C.c_int, [P, C.c_int, p, p, p, p, p]),
            "fpb_host_max_threshold_mask": (C.c_int, [P, p, p, u64p]),
            "fpb_host_compress_indices": (C.c_int, [P, p, p, p]),
            "fpb_host_block_sparse_attention": (C.c_int, [P, C.c_int, p, p, p, p, p, C.c_int, p,
                                                          p, u64p]),
            "fpb_host_dense_attention": (C.c_int, [P, C.c_int, p, p, p, C.c_int, p, p]),
            "fpb_host_prefill": (C.c_int, [P, C.c_int, p, p, p, C.c_int, p, p, p, p, u64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().fpb_last_error().decode(errors="replace")
