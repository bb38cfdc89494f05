"""Far-field order K variants (development aid): timing, pair counts and accuracy against a
saved exact result.  python order_ab.py <cfg> <nq> lib_a.so lib_b.so ..."""
import os, subprocess, sys
if sys.argv[1] == "--child":
    sys.path.insert(0, '.')
    import time
    import numpy as np, torch
    import paper_2408_04466_b200 as G
    from paper_2408_04466_b200 import scenes
    cfg, nq, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    s = scenes.make(cfg, nq)
    t0 = time.perf_counter(); sc = G.Scene(s.ctrl); torch.cuda.synchronize(); tb = time.perf_counter() - t0
    q = torch.from_numpy(s.queries).cuda()
    w, st = G.winding_numbers(sc, q)
    w, st = G.winding_numbers(sc, q)
    sc.set_timing(True)
    w, st = G.winding_numbers(sc, q)
    t = sc.stats()
    tot = t['ms_cull'] + t['ms_intersect'] + t['ms_boundary'] + t['ms_other']
    print(f"{os.path.basename(out)}: scene {tb:.2f}s total={tot:.2f} k4={t['ms_boundary']:.2f} far={t['ms_k4_far']:.2f} exact={t['ms_k4_exact']:.2f} "
          f"far_pairs={t['far_pairs']} terms/pair={t['far_terms']/max(1,t['far_pairs']):.0f} near_pairs={t['near_pairs']} segs={t['boundary_segments']}", flush=True)
    np.savez(out, w=w.cpu().numpy(), st=st.cpu().numpy())
    sys.exit(0)
import numpy as np
cfg, nq, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
if int(nq) <= (1 << 20):
    subprocess.run([sys.executable, __file__, "--child", cfg, nq, "/tmp/ord_exact.npz"], env={**os.environ, "GWN_FARFIELD": "0"})
for lib in libs:
    env = dict(os.environ)
    if lib != "default":
        env["GWN_B200_LIB"] = os.path.abspath(lib)
    out = f"/tmp/ord_{os.path.basename(lib)}.npz"
    subprocess.run([sys.executable, __file__, "--child", cfg, nq, out], env=env)
    if int(nq) <= (1 << 20):
        e, b = np.load("/tmp/ord_exact.npz"), np.load(out)
        ok = (e["st"] == 0) & (b["st"] == 0)
        print("   status equal", np.array_equal(e["st"], b["st"]), "max|dw| vs exact", np.abs(e["w"] - b["w"])[ok].max())
