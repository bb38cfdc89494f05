"""Triangle meshes on the B200 kernels (the reference's surfaces.py:66-431
mesh side): a Morton-order BVH in the array layout of the reference's ``Bvh``
(surfaces.py:74-89, so reference ``Bvh`` objects and these are
interchangeable; the tree itself is built differently, see ``build_bvh``), all-hits
ray/mesh records (``intersect_ray_mesh``, surfaces.py:299-329) and mesh
generalized winding numbers as solid-angle sums (the reference's ground
truth, _kernels.py:385-475) through libgwn_b200.so.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _kernels
from .config import DEFAULT_EPS, EpsilonConfig
from .geometry import Ray
from .surfaces import IntersectionRecord


@dataclass
class Bvh:
    node_min: np.ndarray
    node_max: np.ndarray
    node_left: np.ndarray
    node_right: np.ndarray
    node_start: np.ndarray
    node_count: np.ndarray
    tri_order: np.ndarray
    V0: np.ndarray
    E1: np.ndarray
    E2: np.ndarray
    NN: np.ndarray
    NH: np.ndarray
    C: np.ndarray
    R2: np.ndarray


def _morton30(c: np.ndarray) -> np.ndarray:
    """30-bit Morton codes of points quantised to a 1024^3 grid over their box."""
    lo, hi = c.min(axis=0), c.max(axis=0)
    ext = np.where(hi > lo, hi - lo, 1.0)
    g = np.clip(((c - lo) / ext * 1024.0).astype(np.int64), 0, 1023)
    code = np.zeros(len(c), np.int64)
    for b in range(10):
        for a in range(3):
            code |= ((g[:, a] >> b) & 1) << (3 * b + (2 - a))
    return code


def build_bvh(vertices, triangles, leaf_size: int = 8) -> Bvh:
    """A BVH in the reference's ``Bvh`` array layout (surfaces.py:74-89: node
    boxes, children, leaf ranges into ``tri_order``, per-triangle
    Moller-Trumbore data), so reference ``Bvh`` objects and these are
    interchangeable.  Built differently: triangles are ordered once along a
    Morton curve of their centroids, then the tree is cut level by level into
    halves of that order (numpy, one pass per level), with node boxes from
    segmented min/max reductions.  Leaves hold <= leaf_size triangles."""
    V = np.ascontiguousarray(vertices, dtype=np.float64)
    T = np.ascontiguousarray(triangles, dtype=np.int64).reshape(-1, 3)
    F = len(T)
    p0, p1, p2 = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    cent = (p0 + p1 + p2) / 3.0
    order = np.argsort(_morton30(cent), kind="stable") if F else np.zeros(0, np.int64)
    bmin = np.minimum(np.minimum(p0, p1), p2)[order]
    bmax = np.maximum(np.maximum(p0, p1), p2)[order]
    lo_l, hi_l, par_l, side_l = [np.zeros(1, np.int64)], [np.full(1, F, np.int64)], \
        [np.full(1, -1, np.int64)], [np.zeros(1, np.int64)]
    lo, hi, base = lo_l[0], hi_l[0], 0
    while True:  # breadth-first: the children of this level's inner nodes
        split = (hi - lo) > leaf_size
        if not split.any():
            break
        ids = base + np.nonzero(split)[0]
        mid = (lo[split] + hi[split]) // 2
        lo = np.stack([lo[split], mid], 1).reshape(-1)
        hi = np.stack([mid, hi[split]], 1).reshape(-1)
        base += len(split)
        lo_l.append(lo); hi_l.append(hi)
        par_l.append(np.repeat(ids, 2)); side_l.append(np.tile([0, 1], len(ids)))
    start = np.concatenate(lo_l)
    count = np.concatenate(hi_l) - start
    parent, side = np.concatenate(par_l), np.concatenate(side_l)
    n = len(start)
    left, right = np.full(n, -1, np.int64), np.full(n, -1, np.int64)
    kid = np.arange(n)
    left[parent[(parent >= 0) & (side == 0)]] = kid[(parent >= 0) & (side == 0)]
    right[parent[(parent >= 0) & (side == 1)]] = kid[(parent >= 0) & (side == 1)]
    inner = left >= 0
    start[inner], count[inner] = 0, 0
    nmin, nmax = np.zeros((n, 3)), np.zeros((n, 3))
    leaf = np.nonzero(~inner & (count > 0))[0]
    if len(leaf):  # leaves partition the Morton order: one segmented reduction
        leaf = leaf[np.argsort(start[leaf])]
        nmin[leaf] = np.minimum.reduceat(bmin, start[leaf], axis=0)
        nmax[leaf] = np.maximum.reduceat(bmax, start[leaf], axis=0)
    for lvl in reversed(range(len(lo_l) - 1)):  # inner nodes bottom-up
        a = sum(len(x) for x in lo_l[:lvl])
        ids = a + np.nonzero(inner[a:a + len(lo_l[lvl])])[0]
        nmin[ids] = np.minimum(nmin[left[ids]], nmin[right[ids]])
        nmax[ids] = np.maximum(nmax[left[ids]], nmax[right[ids]])
    e1, e2 = p1 - p0, p2 - p0
    nrm = np.cross(e1, e2)
    nn = np.sqrt((nrm * nrm).sum(axis=1))
    nh = nrm / np.where(nn > 0, nn, 1.0)[:, None]
    r2 = np.max(np.stack([((p - cent) ** 2).sum(axis=1) for p in (p0, p1, p2)]), axis=0)
    return Bvh(nmin, nmax, left, right, start, count, order.astype(np.int64),
               np.ascontiguousarray(p0), np.ascontiguousarray(e1), np.ascontiguousarray(e2),
               np.ascontiguousarray(nn), np.ascontiguousarray(nh), np.ascontiguousarray(cent),
               np.ascontiguousarray(r2))


def intersect_ray_mesh(vertices, triangles, ray: Ray, t_window=(0.0, np.inf),
                       eps: EpsilonConfig = DEFAULT_EPS, bvh: Bvh | None = None
                       ) -> list[IntersectionRecord]:
    """All hits in the window, ascending in t (surfaces.py:299-329)."""
    t_lo, t_hi = t_window
    if t_lo < 0.0:
        raise ValueError("t window must start at 0 or later")
    V = np.asarray(vertices, np.float64)
    bvh = bvh if bvh is not None else build_bvh(V, triangles)
    diag = float(np.linalg.norm(V.max(axis=0) - V.min(axis=0))) if len(V) else 0.0
    plane_tol = 1e-10 * (1.0 + diag)
    ts, tris, dd, us, vs = _kernels.bvh_ray_all_hits(bvh, ray.origin, ray.direction, t_lo, t_hi,
                                                     eps.tangent_parametric, plane_tol)
    recs = []
    for k in np.argsort(ts, kind="stable"):
        f = int(tris[k])
        d = float(dd[k])
        recs.append(IntersectionRecord(
            t=float(ts[k]), point=ray.at(float(ts[k])), normal=bvh.NH[f].copy(),
            sign=1 if d > 0 else -1, tangency=bool(abs(d) <= eps.tangent_parametric),
            grazing=bool(min(us[k], vs[k], 1.0 - us[k] - vs[k]) < eps.edge_graze)))
    return recs


def mesh_winding_numbers(vertices, triangles, points, guard: float = 1e-12):
    """Generalized winding numbers of a triangle soup at many points: the
    solid-angle sum / 4 pi (_kernels.py:466-475) and the on-surface flags."""
    out, on = _kernels.solid_angle_many(vertices, triangles, points, guard)
    return out / (4.0 * np.pi), on
