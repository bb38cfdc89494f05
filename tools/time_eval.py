"""Per-stage timing of one config (development aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes

for arg in sys.argv[1:] or ["2"]:
    cfg, _, nq = arg.partition(":")
    s = scenes.make(int(cfg), int(nq) if nq else None)
    sc = G.Scene(s.ctrl)
    q = torch.from_numpy(s.queries).cuda()
    w, st = G.winding_numbers(sc, q)
    torch.cuda.synchronize()
    t = time.perf_counter(); n = 5
    for _ in range(n):
        w, st = G.winding_numbers(sc, q)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / n
    sc.set_timing(True)
    G.winding_numbers(sc, q)
    stt = sc.stats()
    print(f"cfg{cfg} Q={len(q)} P={sc.n_patches} segs={sc.n_net_segments}: {dt*1e3:.3f} ms/eval "
          f"({len(q)/dt/1e6:.1f} Mq/s) stages cull={stt['ms_cull']:.3f} int={stt['ms_intersect']:.3f} "
          f"bnd={stt['ms_boundary']:.3f} fin={stt['ms_other']:.3f} [k3 cand={stt['ms_k3_candidates']:.3f} "
          f"fb={stt['ms_k3_fallback']:.3f} ({stt['k3_fallback_items']} items) newton={stt['ms_k3_newton']:.3f}] | cand={stt['candidates']} "
          f"nodes={stt['nodes']} newton={stt['newton_iters']} roots={stt['roots']} retried={stt['retried']} "
          f"status={np.unique(st.cpu().numpy(), return_counts=True)}", flush=True)
