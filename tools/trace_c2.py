"""Host-side timeline of gwn_eval on config 2 (GWN_TRACE marks) plus event timing."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
sc = G.Scene(s.ctrl)
q = torch.from_numpy(s.queries).cuda()
w = torch.empty(len(q), dtype=torch.float64, device="cuda"); st = torch.empty(len(q), dtype=torch.int8, device="cuda")
for _ in range(5):
    G.winding_numbers(sc, q, out=(w, st))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in range(3):
    a.record(); t = time.perf_counter()
    G.winding_numbers(sc, q, out=(w, st))
    b.record(); torch.cuda.synchronize()
    print(f"eval: events {a.elapsed_time(b)*1e3:.1f} us, host {(time.perf_counter()-t)*1e6:.1f} us", file=sys.stderr, flush=True)
