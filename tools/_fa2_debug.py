import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2603_06199_b200 as fp
from oracle import Oracle
from tests._util import composite_np, bf16_round
port = Oracle("port")
Z, H, L = 1, 3, 4096
q, k, v = (bf16_round(x) for x in composite_np(13, Z, H, H, L))
tau = float(port.scale(128))
M = L // 128
rng = np.random.default_rng(0)
idx = np.full((Z, M, M, H), M, np.int32)
counts = np.zeros((Z, M, H), np.int32)
for h in range(H):
    for i in range(M):
        if rng.random() < 0.3:
            js = np.sort(rng.choice(i + 1, size=min(i + 1, int(rng.integers(1, 20))), replace=False))
            idx[0, i, :len(js), h] = js
            counts[0, i, h] = len(js)
ro, rl, _ = port.block_sparse_attention(q, k, v, idx, counts, 128, tau)
cu = lambda x, dt=torch.bfloat16: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)
for it in range(10):
  res = fp.block_sparse_attention(cu(q), cu(k), cu(v), fp.SparseBlockPlan(cu(idx, torch.int32), cu(counts, torch.int32)), fp.make_block_grid(L, 128), tau, out_dtype=torch.float32)
  go = res.out.cpu().numpy(); gl = res.lse.cpu().numpy()
  print("iter", it, flush=True)
  for h in range(H):
    for i in range(M):
      c = counts[0, i, h]
      if c == 0: continue
      e = np.abs(go[0, h, i*128:(i+1)*128] - ro[0, h, i*128:(i+1)*128])
      el = np.abs(gl[0, h, i*128:(i+1)*128] - rl[0, h, i*128:(i+1)*128])
      if e.max() > 0.02 or el.max() > 0.02:
        bad_rows = np.where(e.max(1) > 0.02)[0]
        print(f"h={h} i={i} C={c} blocks={idx[0,i,:c,h].tolist()} diag={i in idx[0,i,:c,h]} maxerr={e.max():.3f} lse_err={el.max():.3f} bad rows {bad_rows[:10].tolist()}..{len(bad_rows)}")
