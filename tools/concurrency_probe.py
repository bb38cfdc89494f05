"""Probe (development aid): does splitting one eval into concurrent evals on
separate streams (host threads) overlap the latency-bound stages?"""
import sys, time, threading
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = scenes.make(cfg)
sc = G.Scene(s.ctrl)
q = torch.from_numpy(s.queries).cuda()
n = len(q)
w = torch.empty(n, dtype=torch.float64, device='cuda')
st = torch.empty(n, dtype=torch.int8, device='cuda')
ref, _ = G.winding_numbers(sc, q)
torch.cuda.synchronize()

def run(k, steps=30):
    streams = [torch.cuda.Stream() for _ in range(k)]
    bounds = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    def job(i, bar):
        a, b = bounds[i]
        for _ in range(steps):
            bar.wait()
            G.winding_numbers(sc, q[a:b], index_base=a, out=(w[a:b], st[a:b]),
                              stream=streams[i].cuda_stream)
            bar.wait()
    for rep in range(2):
        bar = threading.Barrier(k + 1)
        ths = [threading.Thread(target=job, args=(i, bar)) for i in range(k)]
        for t in ths: t.start()
        tot = 0.0
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bar.wait()
            bar.wait()
            torch.cuda.synchronize()
            tot += time.perf_counter() - t0
        for t in ths: t.join()
    ok = torch.equal(w, ref)
    print(f"k={k}: {tot / steps * 1e3:.4f} ms/step (wall) bitwise={ok}", flush=True)

for k in (1, 2, 3, 4):
    run(k)
