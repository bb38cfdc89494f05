"""Scene creation (K1 round 0) time per config (development aid)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
torch.cuda.init()
G.Scene(scenes.make(1, 8).ctrl)  # warm the context
for c in (1, 2, 3, 4, 5):
    s = scenes.make(c, 8)
    t = time.perf_counter()
    sc = G.Scene(s.ctrl)
    torch.cuda.synchronize()
    print(f"cfg{c} P={len(s.ctrl)} scene create {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
