"""Ray reuse vs per-point evaluation on voxel grids (development aid).

usage: python tools/time_rays.py CFG:N [CFG:N ...]
Voxelizes the scene AABB at N^3 through gwn_eval_rays (N^2 rays) and times it
against gwn_eval of the same N^3 points (host buffers on both sides).
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2408_04466_b200 as G  # noqa: E402
from paper_2408_04466_b200 import scenes  # noqa: E402


def main():
    for arg in sys.argv[1:] or ["4:128"]:
        cfg, _, n = arg.partition(":")
        n = int(n)
        s = scenes.make(int(cfg), 16)
        sc = G.Scene(s.ctrl)
        bb = sc.aabb()
        c = (np.arange(n) + 0.5) / n
        ax = [bb.min_corner[k] + c * (bb.max_corner[k] - bb.min_corner[k]) for k in range(3)]
        X, Y, Z = np.meshgrid(*ax, indexing="ij")
        pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
        G.voxelize(sc, n)
        G.winding_numbers(sc, pts)
        import torch
        dev = torch.device("cuda")
        cc = (torch.arange(n, dtype=torch.float64, device=dev) + 0.5) / n
        Yd, Zd = torch.meshgrid(torch.as_tensor(ax[1], device=dev), torch.as_tensor(ax[2], device=dev),
                                indexing="ij")
        org = torch.stack([torch.full_like(Yd, bb.min_corner[0]), Yd, Zd], -1).reshape(-1, 3)
        tsd = (cc * (bb.max_corner[0] - bb.min_corner[0])).repeat(n * n)
        offd = torch.arange(n * n + 1, dtype=torch.int64, device=dev) * n
        qd = torch.from_numpy(pts).to(dev)
        for _ in range(2):
            G.winding_numbers_rays(sc, org, [1.0, 0, 0], tsd, offd, check=False)
            G.winding_numbers(sc, qd)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            G.winding_numbers_rays(sc, org, [1.0, 0, 0], tsd, offd, check=False)
        torch.cuda.synchronize()
        trd = (time.perf_counter() - t) / 3
        t = time.perf_counter()
        for _ in range(3):
            G.winding_numbers(sc, qd)
        torch.cuda.synchronize()
        tpd = (time.perf_counter() - t) / 3
        print(f"  device-resident: rays {trd*1e3:.2f} ms ({n**3/trd/1e6:.1f} Mpts/s) vs per-point "
              f"{tpd*1e3:.2f} ms ({n**3/tpd/1e6:.1f} Mpts/s) -> {tpd/trd:.2f}x", flush=True)
        reps = 3
        t = time.perf_counter()
        for _ in range(reps):
            occ, w = G.voxelize(sc, n)
        tr = (time.perf_counter() - t) / reps
        st_r = sc.stats()
        t = time.perf_counter()
        for _ in range(reps):
            wp, sp = G.winding_numbers(sc, pts)
        tp = (time.perf_counter() - t) / reps
        st_p = sc.stats()
        m = sp == 0
        d = np.abs(w.ravel() - wp)[m].max() if m.any() else 0.0
        print(f"cfg{cfg} N={n} pts={n**3} P={sc.n_patches}: rays {tr*1e3:.1f} ms "
              f"({n**3/tr/1e6:.1f} Mpts/s, {sc.rays_cast} rays, cand={st_r['candidates']} "
              f"retried={st_r['retried']}) | per-point {tp*1e3:.1f} ms ({n**3/tp/1e6:.1f} Mpts/s, "
              f"cand={st_p['candidates']}) | speedup {tp/tr:.2f}x maxdiff {d:.2e}", flush=True)


if __name__ == "__main__":
    main()
