"""A/B of the two K4 kernels (GWN_K4_GENERIC): bit-identity and time (development aid)."""
import os, subprocess, sys, json
sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch
    import paper_2408_04466_b200 as G
    from paper_2408_04466_b200 import scenes
    out = {}
    for cfg, nq in ((1, 4096), (3, 1 << 18), (5, 1 << 15)):
        s = scenes.make(cfg, nq)
        sc = G.Scene(s.ctrl)
        q = torch.from_numpy(s.queries).cuda()
        w, st = G.winding_numbers(sc, q)
        torch.cuda.synchronize()
        sc.set_timing(True)
        G.winding_numbers(sc, q)
        ms = sc.stats()["ms_boundary"]
        sc.set_timing(False)
        np.save(f"/tmp/k4_{cfg}_{os.environ.get('GWN_K4_GENERIC', '0')}.npy", w.cpu().numpy())
        out[cfg] = ms
    print(json.dumps(out))
else:
    res = {}
    for gen in ("0", "1"):
        env = dict(os.environ)
        if gen == "1":
            env["GWN_K4_GENERIC"] = "1"
        else:
            env.pop("GWN_K4_GENERIC", None)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        res[gen] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
    print("edge-aligned ms:", res["0"], " generic ms:", res["1"])
    import numpy as np
    for cfg in (1, 3, 5):
        a, b = np.load(f"/tmp/k4_{cfg}_0.npy"), np.load(f"/tmp/k4_{cfg}_1.npy")
        print(cfg, "bit-identical" if np.array_equal(a, b) else f"DIFF max {np.abs(a-b).max()}")
