"""Device-resident vs host-buffer (pinned, pipelined) eval of a config, wall clock (development aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nq = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 26)
s = scenes.make(cfg, nq)
sc = G.Scene(s.ctrl)
q_dev = torch.from_numpy(s.queries).cuda()
q_pin = torch.from_numpy(s.queries).pin_memory()
w_dev = torch.empty(nq, dtype=torch.float64, device="cuda"); st_dev = torch.empty(nq, dtype=torch.int8, device="cuda")
w_pin = torch.empty(nq, dtype=torch.float64).pin_memory(); st_pin = torch.empty(nq, dtype=torch.int8).pin_memory()
for name, q, out in (("device", q_dev, (w_dev, st_dev)), ("host", q_pin, (w_pin, st_pin)), ("device", q_dev, (w_dev, st_dev)), ("host", q_pin, (w_pin, st_pin))):
    for i in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        G.winding_numbers(sc, q, out=out)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"{name} {i}: {dt*1e3:.1f} ms  {nq/dt/1e6:.1f} Mq/s", flush=True)
