"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the builder container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
writes small .npz fixtures next to this script.  The fixtures travel with the
repo; nothing at test time reads /root/reference.

What is captured (reference file:line):
  clip.npz      gwn.geometry.ray_aabb_clip                  geometry.py:198-219
  boundary.npz  gwn.surfaces.patch_boundary via a bicubic adapter of the
                reference patch protocol                    surfaces.py:611-626
  roots.npz     gwn.surfaces._multistart_ray_roots, as shipped (whole patch)
                and run on 8x8 de Casteljau sub-patches,
                plus a dense-tessellation hit count through the numpy twin
                _ray_tris_hits_numpy                         surfaces.py:634-701,
                                                            _kernels.py:312-363
  fan.npz       gwn._kernels.single_loop_batch from a scratch copy with the
                one-line _cross fix (_kernels.py:45), as-shipped output too
                                                            _kernels.py:723-823
  tess.npz      dense-tessellation w through _solid_angle_numpy
                                                            _kernels.py:422-440
  scene3.npz,   scene-level sums of the reference's per-patch terms: for each
  scene5.npz    query and patch, chi from the reference solver on de
                Casteljau sub-patches and w_k = single_loop_batch(loop_k,
                hits_k) from the line-45-fixed copy (chi + the fan formula
                where it returns ok = 0, counted in `fallback`); w = sum_k
                w_k (SPEC additivity).  Config 3 (64 patches) and
                config 5 (15,876 patches): pins net-boundary cancellation,
                the far field and re-shoot-free round-0 values against the
                reference.                                   surfaces.py:611-701,
                                                            _kernels.py:723-823

    python tests/golden/make_golden.py scene    # only the scene fixtures
"""

from __future__ import annotations

import importlib
import math
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REPO)

from paper_2408_04466_b200 import scenes  # noqa: E402  (seeded generators)

sys.path.insert(0, REF_SRC)
import gwn.geometry as G  # noqa: E402
import gwn.surfaces as SU  # noqa: E402
from gwn.config import DEFAULT_EPS  # noqa: E402

DIR_SEED = 0x2408044660


# ---------------------------------------------------------------------------
# bicubic adapter of the reference patch protocol (template CoonsPatch,
# surfaces.py:499-589).  No bicubic type exists in the reference.
# ---------------------------------------------------------------------------


def _b(t):
    s = 1.0 - t
    return np.array([s ** 3, 3 * t * s * s, 3 * t * t * s, t ** 3])


def _db(t):
    s = 1.0 - t
    return np.array([-3 * s * s, 3 * s * s - 6 * t * s, 6 * t * s - 3 * t * t, 3 * t * t])


class BicubicAdapter:
    def __init__(self, ctrl, patch_id=0, parent=None):
        self.control = np.ascontiguousarray(ctrl, dtype=np.float64).reshape(4, 4, 3)
        self.patch_id = patch_id
        self.may_self_intersect = False
        self.parent = parent          # (u0, v0, w) when this is a sub-patch

    def point(self, u, v):
        return np.einsum("i,j,ijk->k", _b(u), _b(v), self.control)

    def partials(self, u, v):
        return (np.einsum("i,j,ijk->k", _db(u), _b(v), self.control),
                np.einsum("i,j,ijk->k", _b(u), _db(v), self.control))

    def aabb(self):
        return G.Aabb.of_points(self.control.reshape(-1, 3))

    def domain_edges(self):
        return [lambda t: (t, 0.0), lambda t: (1.0, t),
                lambda t: (1.0 - t, 1.0), lambda t: (0.0, 1.0 - t)]

    def domain_contains(self, u, v, tol):
        return -tol <= u <= 1.0 + tol and -tol <= v <= 1.0 + tol

    def domain_boundary_dist(self, u, v):
        if self.parent is not None:   # grazing measured in the parent domain
            u0, v0, w = self.parent
            u, v = u0 + w * u, v0 + w * v
        return min(u, 1.0 - u, v, 1.0 - v)

    def domain_center(self):
        return (0.5, 0.5)


def split(net, axis):
    """de Casteljau halving of a (4,4,3) net along axis 0 (u) or 1 (v)."""
    n = np.moveaxis(net, axis, 0)
    p0, p1, p2, p3 = n
    a01, a12, a23 = (p0 + p1) / 2, (p1 + p2) / 2, (p2 + p3) / 2
    b0, b1 = (a01 + a12) / 2, (a12 + a23) / 2
    c = (b0 + b1) / 2
    left = np.stack([p0, a01, b0, c])
    right = np.stack([c, b1, a23, p3])
    return np.moveaxis(left, 0, axis), np.moveaxis(right, 0, axis)


def sub_patches(ctrl, depth):
    out = [(np.asarray(ctrl, dtype=np.float64), 0.0, 0.0, 1.0)]
    for _ in range(depth):
        nxt = []
        for net, u0, v0, w in out:
            a, b = split(net, 0)
            h = w / 2
            for half, uu in ((a, u0), (b, u0 + h)):
                c, d = split(half, 1)
                nxt.append((c, uu, v0, h))
                nxt.append((d, uu, v0 + h, h))
        out = nxt
    return out


def ref_hits(patch, o, d):
    ray = G.Ray(np.asarray(o, float), np.asarray(d, float))
    return SU._multistart_ray_roots(patch, ray, DEFAULT_EPS, (0.0, np.inf),
                                    DEFAULT_EPS.tangent_parametric)


def ref_hits_subdivided(ctrl, o, d, depth=3):
    """Reference solver on de Casteljau sub-patches, roots unioned with the
    reference's own 1e-9 dedup rule (surfaces.py:673)."""
    recs = []
    for net, u0, v0, w in sub_patches(ctrl, depth):
        for r in ref_hits(BicubicAdapter(net, parent=(u0, v0, w)), o, d):
            if any(abs(r.t - q.t) < DEFAULT_EPS.dedup for q in recs):
                continue
            recs.append(r)
    recs.sort(key=lambda r: r.t)
    return recs


def tess_mesh(ctrl, n):
    g = np.linspace(0.0, 1.0, n + 1)
    P = np.array([[BicubicAdapter(ctrl).point(u, v) for v in g] for u in g]).reshape(-1, 3)
    T = []
    for i in range(n):
        for j in range(n):
            a, b = i * (n + 1) + j, (i + 1) * (n + 1) + j
            T.append((a, b, b + 1))
            T.append((a, b + 1, a + 1))
    return P, np.asarray(T, np.int64)


def direction(r):
    """Same generator as oracle/gwn_oracle.c or_direction (splitmix64)."""
    M = (1 << 64) - 1

    def sm(s):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return s, z ^ (z >> 31)

    s = DIR_SEED ^ ((0xD1B54A32D192ED03 * (r + 1)) & M)
    s, h1 = sm(s)
    s, h2 = sm(s)
    z = 1.0 - 2.0 * ((h1 >> 11) * (1.0 / 9007199254740992.0))
    phi = 2.0 * math.pi * ((h2 >> 11) * (1.0 / 9007199254740992.0))
    rr = math.sqrt(max(0.0, 1.0 - z * z))
    return np.array([rr * math.cos(phi), rr * math.sin(phi), z])


# ---------------------------------------------------------------------------


def gen_clip(rng):
    n = 400
    lo = rng.uniform(-1, 1, (n, 3))
    hi = lo + rng.uniform(0, 2, (n, 3))
    o = rng.uniform(-3, 3, (n, 3))
    d = rng.normal(size=(n, 3))
    d[::7, 0] = 0.0                     # exact zero components (geometry.py:207-210)
    d[::11, 1] = 0.0
    o[::5] = 0.5 * (lo[::5] + hi[::5])  # origins inside the box
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t = np.full((n, 2), np.nan)
    for k in range(n):
        r = G.ray_aabb_clip(G.Ray(o[k], d[k]), G.Aabb(lo[k], hi[k]))
        if r is not None:
            t[k] = r
    np.savez_compressed(os.path.join(HERE, "clip.npz"), o=o, d=d, lo=lo, hi=hi, t=t)


def gen_boundary():
    out = {}
    pats = {"c1": scenes.config1(8).ctrl[0], "c3": scenes.config3(8).ctrl[9],
            "c4": scenes.config4(8).ctrl[100]}
    for name, ctrl in pats.items():
        for S in (2, 3, 200):
            loop = SU.patch_boundary(BicubicAdapter(ctrl), S)
            out[f"{name}_S{S}"] = loop.points
        out[f"{name}_ctrl"] = ctrl
    np.savez_compressed(os.path.join(HERE, "boundary.npz"), **out)


def gen_roots(rng):
    from gwn import _kernels as K
    K_np = K._ray_tris_hits_numpy
    pats = [scenes.config1(8).ctrl[0], scenes.config2(8).ctrl[4], scenes.config4(8).ctrl[7]]
    rows = []   # patch, ray id, o, d, shipped hits, subdivided hits, tess count
    O, D, PID = [], [], []
    ship, subd, tess_chi = [], [], []
    for pi, ctrl in enumerate(pats):
        lo, hi = ctrl.reshape(-1, 3).min(0), ctrl.reshape(-1, 3).max(0)
        cen, ext = 0.5 * (lo + hi), (hi - lo)
        V, T = tess_mesh(ctrl, 256)
        bvh = SU.build_bvh(V, T)
        for k in range(120):
            o = cen + (rng.uniform(size=3) - 0.5) * ext * 2.0
            # aim most rays at the patch so they hit
            tgt = BicubicAdapter(ctrl).point(*rng.uniform(0.02, 0.98, 2))
            d = tgt - o if k % 4 else rng.normal(size=3)
            d /= np.linalg.norm(d)
            s1 = [(r.t, r.sign, int(r.tangency), int(r.grazing), *r.normal)
                  for r in ref_hits(BicubicAdapter(ctrl), o, d)]
            s2 = [(r.t, r.sign, int(r.tangency), int(r.grazing), *r.normal)
                  for r in ref_hits_subdivided(ctrl, o, d)]
            ts, tris, dd, us, vs = K_np(bvh.V0, bvh.E1, bvh.E2, bvh.NN, bvh.NH, bvh.C, bvh.R2,
                                        o, d, 0.0, np.inf, 1e-12, 1e-10)
            O.append(o); D.append(d); PID.append(pi)
            ship.append(s1); subd.append(s2)
            tess_chi.append(int(np.sum(np.where(dd > 0, 1, -1))) if len(ts) else 0)
    def pack(lst):
        n = np.array([len(x) for x in lst], np.int64)
        flat = np.array([r for x in lst for r in x], np.float64).reshape(-1, 7)
        return n, flat
    sn, sf = pack(ship)
    bn, bf = pack(subd)
    np.savez_compressed(os.path.join(HERE, "roots.npz"), ctrl=np.asarray(pats), pid=np.asarray(PID),
                        o=np.asarray(O), d=np.asarray(D), ship_n=sn, ship=sf, sub_n=bn, sub=bf,
                        tess_chi=np.asarray(tess_chi))


def fixed_kernels():
    """Import gwn._kernels from a scratch copy with the _cross fix (:45)."""
    tmp = tempfile.mkdtemp(prefix="gwnfix_")
    dst = os.path.join(tmp, "gwn_fixed")
    shutil.copytree(os.path.join(REF_SRC, "gwn"), dst,
                    ignore=shutil.ignore_patterns("__pycache__"))
    path = os.path.join(dst, "_kernels.py")
    src = open(path).read()
    bad = "return ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bz"
    assert src.count(bad) == 1, "reference _cross line changed"
    open(path, "w").write(src.replace(bad, "return ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bx"))
    sys.path.insert(0, tmp)
    return importlib.import_module("gwn_fixed._kernels")


def gen_fan(rng):
    from gwn import _kernels as K_ship
    K_fix = fixed_kernels()
    sc = scenes.config1(400)
    ctrl = sc.ctrl[0]
    loop = SU.patch_boundary(BicubicAdapter(ctrl), 200).points
    Q = sc.queries
    dirs = np.array([direction(0), direction(1)])
    w = np.zeros((2, len(Q)))
    ok = np.zeros((2, len(Q)), np.int8)
    w_ship = np.zeros((2, len(Q)))
    ok_ship = np.zeros((2, len(Q)), np.int8)
    chi = np.zeros((2, len(Q)), np.int64)
    for di, d in enumerate(dirs):
        for k, p in enumerate(Q):
            recs = ref_hits_subdivided(ctrl, p, d)
            hts = np.array([r.t for r in recs], float)
            hs = np.array([r.sign for r in recs], np.int64)
            chi[di, k] = int(hs.sum()) if len(hs) else 0
            a, b = K_fix.single_loop_batch(loop, p, d, hts, hs, np.zeros(1), 1e-9, 1e-12)
            w[di, k], ok[di, k] = a[0], b[0]
            a, b = K_ship.single_loop_batch(loop, p, d, hts, hs, np.zeros(1), 1e-9, 1e-12)
            w_ship[di, k], ok_ship[di, k] = a[0], b[0]
    np.savez_compressed(os.path.join(HERE, "fan.npz"), ctrl=ctrl, loop=loop, queries=Q, dirs=dirs,
                        w=w, ok=ok, chi=chi, w_ship=w_ship, ok_ship=ok_ship)


def gen_tess():
    from gwn import _kernels as K
    sc = scenes.config1(600)
    ctrl = sc.ctrl[0]
    V, T = tess_mesh(ctrl, 384)
    keep = []
    for p in sc.queries:
        dist = np.min(np.linalg.norm(V - p, axis=1))
        if dist > 0.05:
            keep.append(p)
        if len(keep) == 150:
            break
    P = np.asarray(keep)
    w = np.array([K._solid_angle_numpy(V, T, p, 1e-12)[0] / (4 * np.pi) for p in P])
    np.savez_compressed(os.path.join(HERE, "tess.npz"), ctrl=ctrl, queries=P, w=w)


def _scene_chunk(args):
    """Worker: per-patch reference terms of a few queries (one ray each along d)."""
    ctrl, loops, Q, d, idx = args
    K_fix = fixed_kernels()
    lo = ctrl.reshape(len(ctrl), -1, 3).min(axis=1)
    hi = ctrl.reshape(len(ctrl), -1, 3).max(axis=1)
    out = []
    for i in idx:
        p = Q[i]
        # patches whose control box the ray meets (the solver's own clip,
        # geometry.py:198-219, vectorised as a prefilter)
        with np.errstate(divide="ignore", invalid="ignore"):
            t0 = (lo - p) / d
            t1 = (hi - p) / d
        tmin = np.where(d != 0, np.minimum(t0, t1), np.where((p >= lo) & (p <= hi), -np.inf, np.inf))
        tmax = np.where(d != 0, np.maximum(t0, t1), np.where((p >= lo) & (p <= hi), np.inf, -np.inf))
        hit = (np.maximum(tmin.max(axis=1), 0.0) <= tmax.min(axis=1))
        w = 0.0
        chi = 0
        fallback = 0
        for k in range(len(ctrl)):
            if hit[k]:
                recs = ref_hits_subdivided(ctrl[k], p, d)
                hts = np.array([r.t for r in recs], float)
                hs = np.array([r.sign for r in recs], np.int64)
            else:
                hts, hs = np.zeros(0), np.zeros(0, np.int64)
            chi += int(hs.sum()) if len(hs) else 0
            a, b = K_fix.single_loop_batch(loops[k], p, d, hts, hs, np.zeros(1), 1e-9, 1e-12)
            if b[0]:
                w += float(a[0])
            else:
                # ok = 0: the reference defers to its (absent) generic path;
                # the fan formula stands in (pinned to this kernel at 1.8e-14
                # where ok = 1, fan.npz)
                from oracle import oracle as O
                w += float(hs.sum() if len(hs) else 0) + O.loop_fan(loops[k], p, d)
                fallback += 1
        out.append((i, w, chi, fallback))
    return out


def gen_scene(cfg, n, nproc=8):
    import multiprocessing as mp
    sc = scenes.make(cfg, n)
    ctrl = np.ascontiguousarray(sc.ctrl)
    loops = [SU.patch_boundary(BicubicAdapter(c), 200).points for c in ctrl]
    d = direction(0)
    Q = sc.queries[:n]
    parts = [list(range(j, n, nproc)) for j in range(nproc)]
    with mp.get_context("fork").Pool(nproc) as pool:
        res = pool.map(_scene_chunk, [(ctrl, loops, Q, d, ix) for ix in parts])
    w = np.zeros(n)
    chi = np.zeros(n, np.int64)
    fb = np.zeros(n, np.int64)
    for part in res:
        for i, wi, ci, fi in part:
            w[i], chi[i], fb[i] = wi, ci, fi
    np.savez_compressed(os.path.join(HERE, f"scene{cfg}.npz"), config=cfg, queries=Q, d=d, w=w,
                        chi=chi, fallback=fb)
    print(f"scene{cfg}.npz: {n} queries, {int(fb.sum())} (query, patch) boundary terms from the "
          f"fan formula where single_loop_batch returned ok = 0")


def main():
    rng = np.random.default_rng(20240804)
    gen_clip(rng)
    gen_boundary()
    gen_roots(rng)
    gen_fan(rng)
    gen_tess()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "scene":
        gen_scene(3, 64)
        gen_scene(5, 16)
    else:
        main()
        gen_scene(3, 64)
        gen_scene(5, 16)
