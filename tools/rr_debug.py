import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
import bench
s = scenes.make(2)
sc = G.Scene(s.ctrl)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
print("alone:", bench.ray_reuse(G, torch, sc, dev, stream, n=256, k=3)["ms"], flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
q = torch.from_numpy(s.queries).to(dev)
for _ in range(5): G.winding_numbers(sc, q)
print("after evals:", bench.ray_reuse(G, torch, sc, dev, stream, n=256, k=3)["ms"], flush=True)
sc.set_timing(True); G.winding_numbers(sc, q); sc.set_timing(False)
print("after timing:", bench.ray_reuse(G, torch, sc, dev, stream, n=256, k=3)["ms"], flush=True)
G.fp64_peak(0)
print("after peak:", bench.ray_reuse(G, torch, sc, dev, stream, n=256, k=3)["ms"], flush=True)
qp = torch.from_numpy(s.queries).pin_memory()
wp = torch.empty(len(qp), dtype=torch.float64).pin_memory()
sp = torch.empty(len(qp), dtype=torch.int8).pin_memory()
for _ in range(3): G.winding_numbers(sc, qp, out=(wp, sp), stream=stream.cuda_stream)
print("after e2e:", bench.ray_reuse(G, torch, sc, dev, stream, n=256, k=3)["ms"], flush=True)
c = bench.ClockSampler(0); c.start(); time.sleep(0.5); m = c.mark(); c.stop(m)
print("after clocks:", bench.ray_reuse(G, torch, sc, dev, stream, n=256, k=3)["ms"], flush=True)
