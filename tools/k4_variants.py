"""Time K4 (far / exact split) across library variants (GWN_B200_LIB) on
config 5 (development aid).  Usage: python tools/k4_variants.py base v1 v2 ..."""
import json
import os
import subprocess
import sys

sys.path.insert(0, ".")
NQ = int(os.environ.get("K4V_QUERIES", 1 << 24))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import paper_2408_04466_b200 as G
    from paper_2408_04466_b200 import scenes
    s = scenes.make(5, NQ)
    sc = G.Scene(s.ctrl)
    q = torch.from_numpy(s.queries).cuda()
    G.winding_numbers(sc, q)
    sc.set_timing(True)
    best = None
    for _ in range(3):
        G.winding_numbers(sc, q)
        t = sc.stats()
        if best is None or t["ms_boundary"] < best["ms_boundary"]:
            best = t
    print(json.dumps({k: round(best[k], 2) for k in ("ms_boundary", "ms_k4_far", "ms_k4_exact")}))
else:
    for v in sys.argv[1:]:
        env = dict(os.environ)
        if v != "base":
            env["GWN_B200_LIB"] = os.path.abspath(f"build/variants/libgwn_b200_{v}.so")
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True,
                           text=True)
        print(v, r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-500:],
              flush=True)
