"""Python-side overhead of winding_numbers (development aid): n = 0 returns in
C before any CUDA call, so the time is the wrapper + ctypes path."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(2, 1024)
sc = G.Scene(s.ctrl)
q = torch.zeros((0, 3), dtype=torch.float64, device='cuda')
w = torch.empty(0, dtype=torch.float64, device='cuda'); st = torch.empty(0, dtype=torch.int8, device='cuda')
strm = torch.cuda.current_stream().cuda_stream
for _ in range(100): G.winding_numbers(sc, q, out=(w, st), stream=strm)
t = time.perf_counter(); n = 20000
for _ in range(n): G.winding_numbers(sc, q, out=(w, st), stream=strm)
print(f"wrapper overhead {1e6 * (time.perf_counter() - t) / n:.2f} us/call")
