"""Minimal driver for ncu: warm-up evals, then one eval between cudaProfilerStart/Stop
(use `ncu --profile-from-start off` to capture only that eval's kernels)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s = scenes.make(cfg, nq or None)
sc = G.Scene(s.ctrl)
q = torch.from_numpy(s.queries).cuda()
for _ in range(2):
    w, st = G.winding_numbers(sc, q)
torch.cuda.synchronize()
torch.cuda.profiler.start()
w, st = G.winding_numbers(sc, q)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", cfg, len(s.queries), sc.stats())
