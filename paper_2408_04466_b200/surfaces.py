"""Bicubic Bezier patches behind the reference patch protocol.

The reference defines the protocol by example (``CoonsPatch``,
pkg/src/gwn/surfaces.py:499-589; ``BezierTrianglePatch`` :431-477):
``point``, ``partials``, ``aabb``, ``domain_edges``, ``domain_contains``,
``domain_boundary_dist``, ``domain_center``, ``boundary_loops``, ``all_hits``
and the ``may_self_intersect`` / ``patch_id`` attributes.  It ships no
bicubic tensor-product type; :class:`BicubicPatch` supplies
one with the same contract.  ``all_hits`` runs on the GPU (the K3 root
enumerator of csrc/gwn_intersect.cu through ``gwn_all_hits``); point /
partial evaluation and boundary sampling are cheap host helpers.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import DEFAULT_EPS, EpsilonConfig
from .errors import DegenerateNormal, OutsideDomain
from .geometry import Aabb, Ray, Vec3


@dataclass(frozen=True)
class IntersectionRecord:
    """One ray-surface hit (surfaces.py:33-48)."""

    t: float
    point: Vec3
    normal: Vec3
    sign: int
    tangency: bool
    grazing: bool = False


@dataclass(frozen=True)
class BoundaryLoop:
    """Closed oriented polyline (surfaces.py:51-65)."""

    points: np.ndarray
    patch_id: int = 0

    def __post_init__(self):
        pts = np.ascontiguousarray(self.points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 3 or pts.shape[0] < 3:
            raise ValueError("a boundary loop needs at least 3 points of shape (N, 3)")
        object.__setattr__(self, "points", pts)

    def reversed(self) -> "BoundaryLoop":
        return BoundaryLoop(self.points[::-1].copy(), self.patch_id)


def _bern(t: float) -> np.ndarray:
    s = 1.0 - t
    return np.array([s * s * s, 3.0 * t * s * s, 3.0 * t * t * s, t * t * t])


def _dbern(t: float) -> np.ndarray:
    s = 1.0 - t
    return np.array([-3.0 * s * s, 3.0 * s * s - 6.0 * t * s, 6.0 * t * s - 3.0 * t * t,
                     3.0 * t * t])


class BicubicPatch:
    """Tensor-product bicubic Bezier patch, control net ``(4, 4, 3)``.

    ``control[i, j]`` with i the u index: f(u,v) = sum B_i(u) B_j(v) P_ij;
    normal f_u x f_v; boundary CCW in (u, v).
    """

    def __init__(self, control, patch_id: int = 0, may_self_intersect: bool = False):
        c = np.ascontiguousarray(control, dtype=np.float64)
        if c.shape != (4, 4, 3):
            raise ValueError("a bicubic patch has a 4x4 net of 3-D control points")
        self.control = c
        self.patch_id = patch_id
        self.may_self_intersect = may_self_intersect
        self._scene = None

    # --- evaluation --------------------------------------------------------
    def point(self, u: float, v: float) -> Vec3:
        return np.einsum("i,j,ijk->k", _bern(u), _bern(v), self.control)

    def partials(self, u: float, v: float) -> tuple[Vec3, Vec3]:
        return (np.einsum("i,j,ijk->k", _dbern(u), _bern(v), self.control),
                np.einsum("i,j,ijk->k", _bern(u), _dbern(v), self.control))

    def aabb(self) -> Aabb:
        # convex-hull property: the patch lies inside its control box
        return Aabb.of_points(self.control.reshape(-1, 3))

    def domain_edges(self):
        # counter-clockwise around the unit square (surfaces.py:566-573)
        return [lambda t: (t, 0.0), lambda t: (1.0, t),
                lambda t: (1.0 - t, 1.0), lambda t: (0.0, 1.0 - t)]

    def domain_contains(self, u: float, v: float, tol: float) -> bool:
        return -tol <= u <= 1.0 + tol and -tol <= v <= 1.0 + tol

    def domain_boundary_dist(self, u: float, v: float) -> float:
        return min(u, 1.0 - u, v, 1.0 - v)

    def domain_center(self):
        return (0.5, 0.5)

    def boundary_loops(self, samples_per_edge: int = 200) -> list[BoundaryLoop]:
        return [patch_boundary(self, samples_per_edge)]

    def flipped(self) -> "BicubicPatch":
        """Reversed orientation (u <-> v transpose)."""
        return BicubicPatch(np.swapaxes(self.control, 0, 1), self.patch_id,
                            self.may_self_intersect)

    # --- GPU all-hits (surfaces.py:587-589 contract) -------------------------
    def _device_scene(self):
        if self._scene is None:
            from .engine import Scene
            self._scene = Scene([self])
        return self._scene

    def all_hits(self, ray: Ray, t_window=(0.0, np.inf),
                 eps: EpsilonConfig = DEFAULT_EPS) -> list[IntersectionRecord]:
        """Every hit of ``ray`` with the patch inside ``t_window``, sorted by t
        (surfaces.py:587-589, body :634-701), from the GPU root enumerator.
        ``eps`` is forwarded to the device (residual, dedup, tangency,
        grazing and degeneracy thresholds).  A near-tangent contact the
        subdivision cannot separate comes back as a tangent record, the
        reference's signal to re-shoot."""
        t_lo, t_hi = t_window
        if t_lo < 0.0:
            raise ValueError("t window must start at 0 or later")
        if not t_lo <= t_hi:
            raise ValueError("empty t window")
        sc = self._device_scene()
        cap = 18  # Bezout: a line meets a bicubic patch at most 2*3*3 times
        t = np.zeros(cap)
        uv = np.zeros(2 * cap)
        sg = np.zeros(cap, np.int32)
        tg = np.zeros(cap, np.int8)
        gz = np.zeros(cap, np.int8)
        flags = C.c_int32(0)
        o = np.ascontiguousarray(ray.origin, dtype=np.float64)
        d = np.ascontiguousarray(ray.direction, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        prm = _lib.params_from_eps(eps)
        n = _lib.check(_lib.lib().gwn_all_hits(
            sc.handle, 0, o.ctypes.data_as(dp), d.ctypes.data_as(dp), C.byref(prm),
            float(t_lo), float(t_hi), t.ctypes.data_as(dp),
            uv.ctypes.data_as(dp), sg.ctypes.data_as(C.POINTER(C.c_int32)),
            tg.ctypes.data_as(C.POINTER(C.c_int8)), gz.ctypes.data_as(C.POINTER(C.c_int8)), cap,
            C.byref(flags)), "gwn_all_hits")
        if n > cap:  # cannot happen below Bezout's bound; never truncate silently
            raise RuntimeError(f"all_hits: {n} roots exceed the {cap}-record buffer")
        out = []
        for k in range(n):
            u, v = uv[2 * k], uv[2 * k + 1]
            fu, fv = self.partials(u, v)
            nrm = np.cross(fu, fv)
            nn = math.sqrt(nrm @ nrm)
            nrm = ray.direction.copy() if nn < eps.degenerate else nrm / nn
            out.append(IntersectionRecord(float(t[k]), ray.at(float(t[k])), nrm, int(sg[k]),
                                          bool(tg[k]), bool(gz[k])))
        return out


def eval_bicubic(patch: BicubicPatch, u: float, v: float,
                 eps: EpsilonConfig = DEFAULT_EPS) -> tuple[Vec3, Vec3]:
    """Point and unit normal at (u, v) (contract of eval_coons, surfaces.py:592-603)."""
    if not (0.0 <= u <= 1.0 and 0.0 <= v <= 1.0):
        raise OutsideDomain("(u, v) outside the unit square")
    p = patch.point(u, v)
    fu, fv = patch.partials(u, v)
    n = np.cross(fu, fv)
    nn = math.sqrt(n @ n)
    if nn < eps.degenerate:
        raise DegenerateNormal(f"degenerate normal at (u, v) = ({u}, {v})")
    return p, n / nn


def patch_boundary(patch, samples_per_edge: int = 200) -> BoundaryLoop:
    """Sample the domain edges CCW into one closed loop (surfaces.py:611-626)."""
    if samples_per_edge < 2:
        raise ValueError("need at least 2 samples per edge")
    pts = []
    for edge in patch.domain_edges():
        for t in np.linspace(0.0, 1.0, samples_per_edge)[:-1]:
            u, v = edge(float(t))
            pts.append(patch.point(u, v))
    return BoundaryLoop(np.asarray(pts), patch.patch_id)
