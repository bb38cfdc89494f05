"""C5 at the full 2^26 queries: scene build, one-shot eval, per-stage stats (development aid)."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nq = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 26)
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # 0: the engine's default
s = scenes.make(cfg, nq)
torch.cuda.init()
G.Scene(scenes.make(1, 8).ctrl)
t = time.perf_counter()
sc = G.Scene(s.ctrl, chunk_queries=chunk)
torch.cuda.synchronize()
print(f"scene create {time.perf_counter()-t:.3f} s  local expansions {sc.local_expansions}", flush=True)
q = torch.from_numpy(s.queries).cuda()
for it in range(3):
    sc.set_timing(it == 2)
    torch.cuda.synchronize()
    t = time.perf_counter()
    w, st = G.winding_numbers(sc, q)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    stt = sc.stats()
    print(f"eval {it}: {dt:.3f} s  {nq/dt/1e6:.2f} Mq/s", flush=True)
print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in stt.items()}, flush=True)
print("status", np.unique(st.cpu().numpy(), return_counts=True), flush=True)
