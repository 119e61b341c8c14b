import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2603_06199_b200 as fp
from paper_2603_06199_b200 import workload
for L in (32768, 131072):
    q, k, v = workload.composite(5, 1, 32, 4, L, device="cuda") if L > 32768 else (x.cuda() for x in workload.qwen3_30b_a3b(L, seed=0))
    plan = fp.discover_select(q, k, fp.PipelineConfig())[0]
    M = plan.counts.shape[1]
    idx = plan.indices[0].permute(2, 0, 1).contiguous()  # h, i, slot
    cnt = plan.counts[0].permute(1, 0).contiguous()      # h, i
    ar = torch.arange(M, device="cuda")
    mask = torch.zeros((32, M, M + 1), dtype=torch.bool, device="cuda")
    live = ar[None, None, :] < cnt[:, :, None]
    hh, ii, ss = torch.nonzero(live, as_tuple=True)
    mask[hh, ii, idx[hh, ii, ss].long()] = True
    mask = mask[:, :, :M]
    def stat(a, b):
        inter = (a & b).sum().item(); uni = (a | b).sum().item(); tot = a.sum().item() + b.sum().item()
        return inter / uni, (tot - uni) / tot  # jaccard, fraction of loads saved by sharing
    # adjacent query blocks, same head
    j1, s1 = stat(mask[:, 0:M-1:2], mask[:, 1:M:2])
    # two heads of the same KV group, same block
    j2, s2 = stat(mask[0::2], mask[1::2])
    print(f"L={L}: adjacent blocks same head: jaccard {j1:.3f}, loads saved {s1:.3f}; "
          f"head pairs same block: jaccard {j2:.3f}, loads saved {s2:.3f}")
