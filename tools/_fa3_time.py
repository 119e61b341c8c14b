import sys, math, torch
sys.path.insert(0, "/root/repo")
import paper_2603_06199_b200 as fp
from paper_2603_06199_b200 import workload
from tools.configs import timed
for L in (32768, 131072):
    q, k, v = workload.composite(5, 1, 32, 4, L, device="cuda")
    r = fp.PrefillRunner(q, k, v, fp.PipelineConfig()).capture()
    r.replay_discover(); torch.cuda.synchronize()
    t = timed(r.replay_attend, reps=5, warm=2)
    print(L, "attn ms", round(t, 3), flush=True)
