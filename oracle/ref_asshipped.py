"""The reference package itself, timed on the host cores -- BENCH
INFRASTRUCTURE ONLY (BASELINE.md §2's CPU baseline plan).

Imported only by bench.py's cpu_baseline leg.  It runs the UNMODIFIED
reference (``baseline/_ref``: ``pip install --no-deps --target baseline/_ref``
of /root/reference/pkg) through its own functions:

  * chi: ``gwn.surfaces._multistart_ray_roots`` (surfaces.py:634-701, scipy
    MINPACK hybr, as shipped) on every patch, through a bicubic adapter of the
    reference patch protocol (CoonsPatch, surfaces.py:499-589; the reference
    ships no bicubic type);
  * boundary term: ``single_loop_batch`` (_kernels.py:801-823) of each patch's
    ``patch_boundary`` loop (surfaces.py:611-626, S = 200) with that patch's
    hits -- from a scratch copy made at run time under /tmp with the one-line
    ``_cross`` fix (_kernels.py:45; the shipped numba helper is wrong, SURVEY
    P4).  Where it returns ok = 0 the oracle's fan term is used instead
    (BASELINE.md §2).

Per query: one ray along the engine's round-0 direction, w = sum over patches
of the per-patch single_loop_batch value (chi + boundary of that patch).  The
rate is reported beside the oracle port's; it is not the target.  Every
query where the as-shipped result differs from the oracle's by more than 1e-6
is adjudicated against a dense tessellation's solid angle (the reference's
own ``_solid_angle_numpy``, _kernels.py:422-440).
"""

from __future__ import annotations

import importlib
import multiprocessing as mp
import os
import shutil
import sys
import tempfile
import time

import numpy as np

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(_REPO, "baseline", "_ref")

_M = {}  # imported reference modules (set in the parent, inherited by forked workers)


def _bern(t):
    s = 1.0 - t
    return np.array([s ** 3, 3 * t * s * s, 3 * t * t * s, t ** 3])


def _dbern(t):
    s = 1.0 - t
    return np.array([-3 * s * s, 3 * s * s - 6 * t * s, 6 * t * s - 3 * t * t, 3 * t * t])


class RefBicubic:
    """Bicubic patch behind the reference patch protocol (the reference's own
    Aabb type, so ray_aabb_clip and the seeding rules run unchanged)."""

    def __init__(self, ctrl, patch_id=0):
        self.control = np.ascontiguousarray(ctrl, dtype=np.float64).reshape(4, 4, 3)
        self.patch_id = patch_id
        self.may_self_intersect = False

    def point(self, u, v):
        return np.einsum("i,j,ijk->k", _bern(u), _bern(v), self.control)

    def partials(self, u, v):
        return (np.einsum("i,j,ijk->k", _dbern(u), _bern(v), self.control),
                np.einsum("i,j,ijk->k", _bern(u), _dbern(v), self.control))

    def aabb(self):
        return _M["geometry"].Aabb.of_points(self.control.reshape(-1, 3))

    def domain_edges(self):
        return [lambda t: (t, 0.0), lambda t: (1.0, t),
                lambda t: (1.0 - t, 1.0), lambda t: (0.0, 1.0 - t)]

    def domain_contains(self, u, v, tol):
        return -tol <= u <= 1.0 + tol and -tol <= v <= 1.0 + tol

    def domain_boundary_dist(self, u, v):
        return min(u, 1.0 - u, v, 1.0 - v)

    def domain_center(self):
        return (0.5, 0.5)


def _load():
    if _M:
        return _M
    if not os.path.isdir(os.path.join(REF_DIR, "gwn")):
        raise FileNotFoundError(f"{REF_DIR}/gwn (pip install --no-deps --target baseline/_ref "
                                "/root/reference/pkg)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    _M["geometry"] = importlib.import_module("gwn.geometry")
    _M["surfaces"] = importlib.import_module("gwn.surfaces")
    _M["config"] = importlib.import_module("gwn.config")
    _M["kernels_shipped"] = importlib.import_module("gwn._kernels")
    # scratch copy with the one-line _cross fix (_kernels.py:45)
    tmp = tempfile.mkdtemp(prefix="gwnref_fix_")
    dst = os.path.join(tmp, "gwn_fixed")
    shutil.copytree(os.path.join(REF_DIR, "gwn"), dst,
                    ignore=shutil.ignore_patterns("__pycache__"))
    path = os.path.join(dst, "_kernels.py")
    src = open(path).read()
    bad = "return ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bz"
    if src.count(bad) != 1:
        raise RuntimeError("reference _cross line changed")
    open(path, "w").write(src.replace(
        bad, "return ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bx"))
    sys.path.insert(0, tmp)
    _M["kernels"] = importlib.import_module("gwn_fixed._kernels")
    return _M


def _eval_one(ctrl, loops, p, d):
    """w(p) by the reference's per-patch functions along direction d;
    returns (w, fallback_patches)."""
    from oracle import oracle as O
    SU, GE, K = _M["surfaces"], _M["geometry"], _M["kernels"]
    eps = _M["config"].DEFAULT_EPS
    ray = GE.Ray(p, d)
    w, fb = 0.0, 0
    for k in range(len(ctrl)):
        recs = SU._multistart_ray_roots(RefBicubic(ctrl[k], k), ray, eps, (0.0, np.inf),
                                        eps.tangent_parametric)
        hts = np.array([r.t for r in recs], np.float64)
        hs = np.array([r.sign for r in recs], np.int64)
        wk, ok = K.single_loop_batch(loops[k], p, d, hts, hs, np.zeros(1), 1e-9, 1e-12)
        if ok[0]:
            w += float(wk[0])
        else:  # generic path: chi + the fan term
            fb += 1
            w += float(hs.sum()) + O.loop_fan(loops[k], p, d)
    return w, fb


def _chunk(args):
    ctrl, loops, Q, d = args
    out = np.empty(len(Q))
    fb = 0
    for i, p in enumerate(Q):
        out[i], f = _eval_one(ctrl, loops, p, d)
        fb += f
    return out, fb


def _tess_w(ctrl, p, n):
    """Solid angle / 4 pi of every patch tessellated at n x n (reference
    _solid_angle_numpy, _kernels.py:422-440)."""
    K = _M["kernels"]
    g = np.linspace(0.0, 1.0, n + 1)
    B = np.stack([_bern(t) for t in g])
    tot = 0.0
    for c in ctrl:
        P = np.einsum("ui,vj,ijk->uvk", B, B, c).reshape(-1, 3)
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        a = (i * (n + 1) + j).ravel()
        b = ((i + 1) * (n + 1) + j).ravel()
        T = np.concatenate([np.stack([a, b, b + 1], 1), np.stack([a, b + 1, a + 1], 1)])
        tot += float(K._solid_angle_numpy(P, T.astype(np.int64), np.asarray(p, np.float64),
                                          1e-12)[0])
    return tot / (4.0 * np.pi)


def measure_config(cfg: int, n: int, cores: int, tess: int = 192) -> dict:
    from oracle import oracle as O
    from paper_2408_04466_b200 import scenes
    _load()
    s = scenes.make(cfg, max(n, 8))
    ctrl, Q = s.ctrl, s.queries[:n]
    d = O.direction(O.params().dir_seed, 0)
    loops = [_M["surfaces"].patch_boundary(RefBicubic(c), 200).points for c in ctrl]
    _chunk((ctrl, loops, Q[:2], d))  # numba compile in the parent (inherited by fork)
    parts = np.array_split(np.arange(n), max(1, cores * 4))
    t = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_chunk, [(ctrl, loops, Q[ix], d) for ix in parts if len(ix)])
    dt = time.perf_counter() - t
    w_ref = np.concatenate([r[0] for r in res])
    fb = sum(r[1] for r in res)
    # the oracle on the same queries and the same (round-0) direction
    chi, bt, fl = O.scene_eval_dir(ctrl, Q, d, nthreads=cores)
    w_or = chi + bt
    clean = fl == 0
    diff = np.abs(w_ref - w_or) > 1e-6
    bad = np.nonzero(diff & clean)[0]
    ref_wrong = orc_wrong = 0
    for i in bad[:16]:  # adjudicate (dense tessellation is slow; at most 16)
        wt = _tess_w(ctrl, Q[i], tess)
        if abs(wt - w_or[i]) < abs(wt - w_ref[i]):
            ref_wrong += 1
        else:
            orc_wrong += 1
    return {"workload": f"first {n} queries of config {cfg} ({len(ctrl)} patches), one ray each "
                        "along the round-0 direction",
            "value": n / dt, "unit": "queries/s", "seconds": dt, "cores": cores,
            "pairs_per_s": n * len(ctrl) / dt,
            "single_loop_batch_fallback_frac": fb / (n * len(ctrl)),
            "disagreements_vs_oracle": int(len(bad)),
            "disagreement_rate": float(len(bad) / max(1, int(clean.sum()))),
            "adjudicated": {"checked": int(min(16, len(bad))), "reference_wrong": ref_wrong,
                            "oracle_wrong": orc_wrong,
                            "judge": f"reference _solid_angle_numpy of a {tess}x{tess} "
                                     "tessellation per patch"}}


def measure(cores: int) -> dict:
    out = {"what": "the reference package as shipped (baseline/_ref): chi by "
                   "_multistart_ray_roots (scipy hybr), boundary by single_loop_batch from a "
                   "run-time scratch copy with the _kernels.py:45 fix; BASELINE.md §2",
           "cpu_model": _cpu_model(), "cores": cores}
    for cfg in (1, 2):
        out[f"config{cfg}"] = measure_config(cfg, 4096, cores)
    return out


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
