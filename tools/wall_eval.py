"""Wall-clock time of warm device-resident evals, per library variant (development aid).
python wall_eval.py cfg[:queries],... lib.so|default ..."""
import os, subprocess, sys, hashlib
if sys.argv[1] != "--child":
    for lib in sys.argv[2:]:
        env = dict(os.environ)
        if lib != "default":
            env["GWN_B200_LIB"] = os.path.abspath(lib)
        print("==", lib, flush=True)
        subprocess.run([sys.executable, __file__, "--child", sys.argv[1]], env=env)
    sys.exit(0)
sys.path.insert(0, ".")
import time
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
for arg in sys.argv[2].split(","):
    cfg, _, nq = arg.partition(":")
    s = scenes.make(int(cfg), int(nq) if nq else None)
    sc = G.Scene(s.ctrl)
    q = torch.from_numpy(s.queries).cuda()
    for _ in range(3):
        w, st = G.winding_numbers(sc, q)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter(); w, st = G.winding_numbers(sc, q); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    h = hashlib.sha1(w.cpu().numpy().tobytes() + st.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"cfg{cfg} Q={len(q)}: best {min(ts)*1e3:.3f} ms median {sorted(ts)[2]*1e3:.3f} ms  {len(q)/min(ts)/1e6:.1f} Mq/s sha={h}", flush=True)
