"""Triangle meshes on the B200 kernels (the reference's surfaces.py:66-431
mesh side): the median-split BVH of ``build_bvh`` (surfaces.py:91-163, same
arrays, so reference ``Bvh`` objects and these are interchangeable), all-hits
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


def build_bvh(vertices, triangles, leaf_size: int = 8) -> Bvh:
    """Median split over triangle centroids along the widest centroid axis
    (surfaces.py:91-163); leaves hold <= leaf_size triangles."""
    V = np.ascontiguousarray(vertices, dtype=np.float64)
    T = np.ascontiguousarray(triangles, dtype=np.int64).reshape(-1, 3)
    F = len(T)
    p0, p1, p2 = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    tmin = np.minimum(np.minimum(p0, p1), p2)
    tmax = np.maximum(np.maximum(p0, p1), p2)
    cent = (p0 + p1 + p2) / 3.0
    nmin, nmax, left, right, start, count = [], [], [], [], [], []
    order = np.arange(F, dtype=np.int64)

    def node():
        nmin.append(np.zeros(3)); nmax.append(np.zeros(3))
        left.append(-1); right.append(-1); start.append(0); count.append(0)
        return len(nmin) - 1

    stack = [(node(), 0, F)]
    while stack:
        nd, lo, hi = stack.pop()
        ids = order[lo:hi]
        nmin[nd] = tmin[ids].min(axis=0) if hi > lo else np.zeros(3)
        nmax[nd] = tmax[ids].max(axis=0) if hi > lo else np.zeros(3)
        if hi - lo <= leaf_size:
            start[nd] = lo
            count[nd] = hi - lo
            continue
        axis = int(np.argmax(cent[ids].max(axis=0) - cent[ids].min(axis=0)))
        mid = (lo + hi) // 2
        order[lo:hi] = ids[np.argsort(cent[ids, axis], kind="stable")]
        a, b = node(), node()
        left[nd], right[nd] = a, b
        stack.append((a, lo, mid))
        stack.append((b, mid, hi))
    e1, e2 = p1 - p0, p2 - p0
    n = np.cross(e1, e2)
    nn = np.linalg.norm(n, axis=1)
    nh = n / np.where(nn > 0, nn, 1.0)[:, None]
    r2 = np.maximum(np.maximum(np.einsum("ij,ij->i", p0 - cent, p0 - cent),
                               np.einsum("ij,ij->i", p1 - cent, p1 - cent)),
                    np.einsum("ij,ij->i", p2 - cent, p2 - cent))
    return Bvh(np.asarray(nmin, np.float64).reshape(-1, 3),
               np.asarray(nmax, np.float64).reshape(-1, 3),
               np.asarray(left, np.int64), np.asarray(right, np.int64),
               np.asarray(start, np.int64), np.asarray(count, np.int64), order,
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
