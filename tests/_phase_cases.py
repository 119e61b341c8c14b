# Cases for tests/test_gpu_phases.py (executed in a child process with FPB_FA_PHASES set).
import math

import torch


def run(fp, case):
    B = 128
    if case == "sparse":  # discovery plan, long enough rows to cross every phase boundary
        q, k, v = fp.workload.composite(3, 1, 4, 2, 40 * B, device="cuda")
        plan = fp.discover_select(q, k, fp.PipelineConfig(alpha=0.1))[0]
    elif case == "ragged_gqa":  # Z = 2, ragged last block, GQA 3:1
        q, k, v = fp.workload.composite(8, 2, 3, 1, 37 * B - 45, device="cuda")
        plan = fp.discover_select(q, k, fp.PipelineConfig(alpha=0.05))[0]
    elif case == "arbitrary":  # random masks incl. j > i, empty rows and empty sub-ranges
        q, k, v = fp.workload.composite(5, 1, 2, 1, 24 * B, device="cuda")
        M = 24
        g = torch.Generator().manual_seed(4)
        mask = (torch.rand((1, M, M, 2), generator=g) < 0.25).to(torch.uint8)
        mask[0, 5] = 0                 # an empty row (C = 0 -> NaN / -inf)
        mask[0, 20, :12] = 0           # a long row with nothing in the first ranges
        mask[0, 21, 8:] = 0            # a long row with nothing in the last ranges
        plan = fp.compress_indices(fp.ActiveMask(mask.cuda()))
    else:
        q, k, v = fp.workload.composite(6, 1, 4, 2, 33 * B, device="cuda")
        plan = None
    L = q.shape[2]
    grid = fp.make_block_grid(L, B)
    tau = 1 / math.sqrt(128)
    if plan is None:
        r = fp.dense_attention(q, k, v, tau, out_dtype=torch.bfloat16)
        return {"out": r.out, "lse": r.lse}
    st = fp.AttentionStats()
    r = fp.block_sparse_attention(q, k, v, plan, grid, tau, st, out_dtype=torch.bfloat16)
    r32 = fp.block_sparse_attention(q, k, v, plan, grid, tau, out_dtype=torch.float32)
    return {"out": r.out, "lse": r.lse, "out32": r32.out, "lse32": r32.lse,
            "visits": torch.tensor([st.block_visits])}
