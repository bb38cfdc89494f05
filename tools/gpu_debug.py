"""Ad-hoc GPU vs oracle comparison printer (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
from oracle import oracle as O

sizes = {1: 4096, 2: 1 << 16, 3: 1 << 14, 4: 1 << 13, 5: 384}
for cfg in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    s = scenes.make(cfg, sizes[cfg])
    t = time.time(); sc = G.Scene(s.ctrl); t_sc = time.time() - t
    w, st = G.winding_numbers(sc, s.queries)
    t = time.time(); w, st = G.winding_numbers(sc, s.queries); t_g = time.time() - t
    stats = sc.stats()
    t = time.time(); wo, so, chi, rounds = O.scene_eval(s.ctrl, s.queries); t_o = time.time() - t
    both = (st == 0) & (so == 0)
    d = np.abs(w - wo)
    print(f"cfg{cfg}: n={len(w)} scene {t_sc*1e3:.1f}ms gpu {t_g*1e3:.1f}ms oracle {t_o:.2f}s "
          f"st_gpu={dict(zip(*np.unique(st, return_counts=True)))} st_or={dict(zip(*np.unique(so, return_counts=True)))} "
          f"max|dw| both-ok={d[both].max() if both.any() else -1:.3e} n_bad(>1e-9)={(d[both]>1e-9).sum()}")
    print("   stats", {k: v for k, v in stats.items() if v})
    bad = np.where(both & (d > 1e-9))[0][:5]
    for b in bad:
        print("   bad", b, s.queries[b], w[b], wo[b], chi[b])
