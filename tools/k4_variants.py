"""Time K4 across library variants (GWN_B200_LIB) on configs 3 and 5 (development aid)."""
import json, os, subprocess, sys
sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch
    import paper_2408_04466_b200 as G
    from paper_2408_04466_b200 import scenes
    out = {}
    for cfg, nq in ((3, 1 << 20), (5, 1 << 15)):
        s = scenes.make(cfg, nq)
        sc = G.Scene(s.ctrl)
        q = torch.from_numpy(s.queries).cuda()
        G.winding_numbers(sc, q)
        sc.set_timing(True)
        t = []
        for _ in range(3):
            G.winding_numbers(sc, q)
            t.append(sc.stats()["ms_boundary"])
        out[cfg] = round(min(t), 3)
    print(json.dumps(out))
else:
    for v in sys.argv[1:]:
        env = dict(os.environ)
        if v != "base":
            env["GWN_B200_LIB"] = os.path.abspath(f"build/variants/libgwn_b200_{v}.so")
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(v, r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-500:], flush=True)
