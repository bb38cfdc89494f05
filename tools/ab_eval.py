"""A/B of library variants (development aid): per-stage timing of configs and a
bitwise comparison of the results across variants.
usage: ab_eval.py cfg[:queries],... lib_a.so lib_b.so ...  (each variant in a fresh process)"""
import os, subprocess, sys, hashlib
if len(sys.argv) > 2 and sys.argv[1] != "--child":
    cfgs, libs = sys.argv[1], sys.argv[2:]
    for lib in libs:
        env = dict(os.environ)
        if lib != "default":
            env["GWN_B200_LIB"] = os.path.abspath(lib)
        print("==", lib, flush=True)
        subprocess.run([sys.executable, __file__, "--child", cfgs], env=env)
    sys.exit(0)
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
for arg in sys.argv[2].split(","):
    cfg, _, nq = arg.partition(":")
    s = scenes.make(int(cfg), int(nq) if nq else None)
    sc = G.Scene(s.ctrl)
    q = torch.from_numpy(s.queries).cuda()
    for _ in range(2):
        w, st = G.winding_numbers(sc, q)
    sc.set_timing(True)
    w, st = G.winding_numbers(sc, q)
    t = sc.stats()
    h = hashlib.sha1(w.cpu().numpy().tobytes() + st.cpu().numpy().tobytes()).hexdigest()[:12]
    tot = t['ms_cull'] + t['ms_intersect'] + t['ms_boundary'] + t['ms_other']
    print(f"cfg{cfg} Q={len(q)}: total={tot:.3f} cull={t['ms_cull']:.3f} cand={t['ms_k3_candidates']:.3f} "
          f"fb={t['ms_k3_fallback']:.3f} newton={t['ms_k3_newton']:.3f} k4={t['ms_boundary']:.3f} "
          f"iters={t['newton_iters']} roots={t['roots']} frac={(t['newton_iters']*220+t['roots']*200)/(t['ms_k3_newton']*1e-3)/34.0e12:.3f} sha={h}", flush=True)
