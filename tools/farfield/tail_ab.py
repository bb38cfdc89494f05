"""A-posteriori order thresholds (GWN_FF_TAIL) vs the a-priori ones and vs the exact K4
(development aid): python tail_ab.py <cfg> <nq>."""
import os, subprocess, sys
if len(sys.argv) > 3:
    sys.path.insert(0, '.')
    import numpy as np, torch
    import paper_2408_04466_b200 as G
    from paper_2408_04466_b200 import scenes
    cfg, nq, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    s = scenes.make(cfg, nq)
    sc = G.Scene(s.ctrl)
    q = torch.from_numpy(s.queries).cuda()
    w, st = G.winding_numbers(sc, q)
    sc.set_timing(True)
    w, st = G.winding_numbers(sc, q)
    t = sc.stats()
    print(f"{out}: k4={t['ms_boundary']:.3f} far={t['ms_k4_far']:.3f} exact={t['ms_k4_exact']:.3f} "
          f"far_pairs={t['far_pairs']} far_terms={t['far_terms']} terms/pair={t['far_terms']/max(1,t['far_pairs']):.1f} "
          f"near_pairs={t['near_pairs']}", flush=True)
    np.savez(out, w=w.cpu().numpy(), st=st.cpu().numpy())
    sys.exit(0)
import numpy as np
cfg, nq = sys.argv[1], sys.argv[2]
runs = {"exact": {"GWN_FARFIELD": "0"}, "apriori": {"GWN_FF_TAIL": "0"}, "tail": {}}
for name, env in runs.items():
    if name == "exact" and int(nq) > (1 << 20):
        continue
    subprocess.run([sys.executable, __file__, cfg, nq, f"/tmp/tail_{name}.npz"], env={**os.environ, **env})
a = np.load("/tmp/tail_apriori.npz"); b = np.load("/tmp/tail_tail.npz")
ok = (a["st"] == 0) & (b["st"] == 0)
print("status equal", np.array_equal(a["st"], b["st"]), "max|dw| tail vs apriori", np.abs(a["w"] - b["w"])[ok].max())
if os.path.exists("/tmp/tail_exact.npz") and int(nq) <= (1 << 20):
    e = np.load("/tmp/tail_exact.npz")
    ok = (e["st"] == 0) & (b["st"] == 0)
    print("max|dw| tail vs exact", np.abs(e["w"] - b["w"])[ok].max(), " apriori vs exact", np.abs(e["w"] - a["w"])[ok & (a['st'] == 0)].max())
