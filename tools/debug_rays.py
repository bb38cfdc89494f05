"""Debug ray-reuse mismatches against per-point eval and the oracle's fixed-direction eval."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2408_04466_b200 as G  # noqa: E402
from paper_2408_04466_b200 import scenes  # noqa: E402
from oracle import oracle as O  # noqa: E402

cfg, n = int(sys.argv[1]), int(sys.argv[2])
s = scenes.make(cfg, 16)
sc = G.Scene(s.ctrl)
bb = sc.aabb()
c = (np.arange(n) + 0.5) / n
ax = [bb.min_corner[k] + c * (bb.max_corner[k] - bb.min_corner[k]) for k in range(3)]
X, Y, Z = np.meshgrid(*ax, indexing="ij")
pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
occ, w = G.voxelize(sc, n)
w = w.ravel()
wp, sp = G.winding_numbers(sc, pts)
bad = np.nonzero((sp == 0) & (np.abs(w - wp) > 1e-9))[0]
print("mismatches", len(bad), "of", len(pts))
d = np.array([1.0, 0.0, 0.0])
if len(bad):
    chi, bt, fl = O.scene_eval_dir(s.ctrl, pts[bad[:50]], d)
    for k, i in enumerate(bad[:20]):
        ix, iy, iz = np.unravel_index(i, (n, n, n))
        print(f"pt {pts[i]} (ix{ix} iy{iy} iz{iz}) ray={w[i]:.12f} pp={wp[i]:.12f} "
              f"oracle_dir chi={chi[k]} b={bt[k]/(2*np.pi):.12f} w={chi[k]+bt[k]/(2*np.pi):.12f} fl={fl[k]}")
    # rays of the first few mismatches: all points along that ray
    i = bad[0]
    ix, iy, iz = np.unravel_index(i, (n, n, n))
    line = np.nonzero((np.arange(n**3) // n) % n == iy)[0]
    sel = [j for j in range(n**3) if np.unravel_index(j, (n, n, n))[1:] == (iy, iz)][:n]
    chi2, bt2, fl2 = O.scene_eval_dir(s.ctrl, pts[sel], d)
    print("ray", iy, iz)
    for j, q in enumerate(sel):
        print(f"  x={pts[q][0]:.6f} ray={w[q]:.9f} pp={wp[q]:.9f} o_chi={chi2[j]} "
              f"o_w={chi2[j]+bt2[j]/(2*np.pi):.9f} fl={fl2[j]}")
    o = np.array([bb.min_corner[0] - 1, pts[i][1], pts[i][2]])
    for p in range(sc.n_patches):
        h = G.BicubicPatch(s.ctrl[p]).all_hits(G.Ray(o, d))
        for r in h:
            print("  hit patch", p, "t", r.t - 1 + bb.min_corner[0], "x", o[0] + r.t, "sign", r.sign)
