"""Config 5 eval time vs chunk size (development aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
nq = int(sys.argv[1])
s = scenes.make(5, nq)
q = torch.from_numpy(s.queries).cuda()
for cq in (0, 1 << 22, 1 << 23):
    sc = G.Scene(s.ctrl, chunk_queries=cq)
    G.winding_numbers(sc, q); torch.cuda.synchronize()
    t = time.perf_counter(); G.winding_numbers(sc, q); torch.cuda.synchronize()
    print(f"chunk {cq}: {1e3 * (time.perf_counter() - t):.1f} ms, segs {sc.stats()['boundary_segments']}", flush=True)
