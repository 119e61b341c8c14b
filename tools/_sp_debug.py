import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2603_06199_b200 as fp
from paper_2603_06199_b200 import workload
for it in range(int(sys.argv[1])):
    q, k, v = workload.composite(5, 1, 32, 4, 2048, device="cuda")
    cfg = fp.PipelineConfig()
    plan = fp.discover_select(q, k, cfg)[0]
    torch.cuda.synchronize()
    res = fp.block_sparse_attention(q, k, v, plan, fp.make_block_grid(2048, 128), cfg.resolved_scale(128))
    torch.cuda.synchronize()
    print("iter", it, "ok", flush=True)
