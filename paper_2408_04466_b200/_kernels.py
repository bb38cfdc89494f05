"""Kernel dispatch layer -- the GPU backend slot of pkg/src/gwn/_kernels.py.

The reference dispatches each hot kernel on ``numba_enabled()``
(_accel.py:28) between a numba and a numpy twin.  Every public kernel of
that module has the same call signature here, backed by libgwn_b200.so:

  single_loop_batch   (:801)  gwn_single_loop_batch
  solid_angle_sum     (:443)  gwn_solid_angle_many (one point)
  solid_angle_many    (:466)  gwn_solid_angle_many
  bvh_ray_all_hits    (:366)  gwn_ray_tris_hits (one ray; ray_tris_hits_batch for R)

arc_crossings (:170) is the generic spherical arrangement's primitive, which
the arrangement-free fan formula supersedes (out of scope); it
has no GPU backend here.

Contiguous float64/int64 in, fresh arrays out, per-element flags instead of
exceptions; the numpy twins' semantics (the numba kernels share the broken
_cross helper, :45).  ``single_loop_batch`` has no numpy twin and returns
``None`` without numba in the reference (:809-810).

Semantics differ only where the reference gives up: the fan formula handles
self-crossing projections and straight edges, so ``ok == 0`` is returned
only for a hit clash (|t_h - t| <= t_eps, :782-784) or a degenerate
projection (:541-542).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def single_loop_batch(loop_pts, origin, direction, hit_ts, hit_signs, query_ts,
                      on_tol, t_eps, device: int = 0):
    loop = np.ascontiguousarray(loop_pts, dtype=np.float64)
    if loop.ndim != 2 or loop.shape[1] != 3 or len(loop) < 3:
        raise ValueError("loop_pts must be (B>=3, 3)")
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(direction, dtype=np.float64)
    ht = np.ascontiguousarray(hit_ts, dtype=np.float64)
    hs = np.ascontiguousarray(hit_signs, dtype=np.int64)
    qt = np.ascontiguousarray(query_ts, dtype=np.float64)
    K = len(qt)
    w = np.zeros(K, np.float64)
    ok = np.zeros(K, np.int8)
    dp = C.POINTER(C.c_double)
    _lib.check(_lib.lib().gwn_single_loop_batch(
        loop.ctypes.data_as(dp), len(loop), o.ctypes.data_as(dp), d.ctypes.data_as(dp),
        ht.ctypes.data_as(dp), hs.ctypes.data_as(C.POINTER(C.c_int64)), len(ht),
        qt.ctypes.data_as(dp), K, float(on_tol), float(t_eps), w.ctypes.data_as(dp),
        ok.ctypes.data_as(C.POINTER(C.c_int8)), device), "gwn_single_loop_batch")
    return w, ok


# ---------------------------------------------------------------------------
# the rest of the dispatch layer (_kernels.py:170, :366, :443, :466); the
# numpy twins' semantics (the numba kernels share the _cross bug, :45)
# ---------------------------------------------------------------------------

def _f64(a, shape=None):
    x = np.ascontiguousarray(a, dtype=np.float64)
    return x.reshape(shape) if shape is not None else x


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def solid_angle_many(V, T, P, guard=1e-12, device: int = 0):
    """Signed solid-angle totals for many query points at once
    (_kernels.py:466-475): ``(out (K,) f64, on_surface (K,) bool)``; ``out``
    is the sum of 2 atan2(num, den), not divided by 4 pi."""
    V = _f64(V, (-1, 3))
    T = _i64(T).reshape(-1, 3)
    P = _f64(P, (-1, 3))
    out = np.empty(len(P), np.float64)
    on = np.zeros(len(P), np.int8)
    _lib.check(_lib.lib().gwn_solid_angle_many(
        _p(V), len(V), _p(T, C.c_int64), len(T), _p(P), len(P), float(guard), _p(out),
        _p(on, C.c_int8), device), "gwn_solid_angle_many")
    return out, on.astype(bool)


def solid_angle_sum(V, T, p, guard=1e-12, device: int = 0):
    """Total signed solid angle of the triangles seen from ``p`` and the
    on-surface flag (_kernels.py:443-451)."""
    out, on = solid_angle_many(V, T, np.asarray(p, np.float64).reshape(1, 3), guard, device)
    return float(out[0]), bool(on[0])


def _bvh_struct(bvh):
    keep = {}

    def arr(name, f):
        a = f(getattr(bvh, name))
        keep[name] = a
        return a.ctypes.data

    b = _lib.TriBvh()
    b.node_min = arr("node_min", lambda x: _f64(x, (-1, 3)))
    b.node_max = arr("node_max", lambda x: _f64(x, (-1, 3)))
    for nm in ("node_left", "node_right", "node_start", "node_count", "tri_order"):
        setattr(b, nm, arr(nm, _i64))
    b.n_nodes = len(keep["node_min"])
    for nm in ("V0", "E1", "E2", "NH", "C"):
        setattr(b, nm, arr(nm, lambda x: _f64(x, (-1, 3))))
    for nm in ("NN", "R2"):
        setattr(b, nm, arr(nm, _f64))
    b.n_tris = len(keep["V0"])
    return b, keep


def ray_tris_hits_batch(bvh, origins, directions, t_lo, t_hi, tang_eps, plane_tol,
                        device: int = 0):
    """All hits of R rays against a reference ``Bvh`` (surfaces.py:74-163):
    CSR ``(offs (R+1,), ts, tris, dotdn, us, vs)``; each ray's hits in the
    numpy twin's order."""
    O = _f64(origins, (-1, 3))
    D = _f64(directions, (-1, 3))
    if O.shape != D.shape:
        raise ValueError("origins and directions must have the same shape")
    b, keep = _bvh_struct(bvh)
    R = len(O)
    offs = np.zeros(R + 1, np.int64)
    cap = 8 * R + 64
    while True:
        ts = np.empty(max(cap, 1)); tris = np.empty(max(cap, 1), np.int64)
        dd = np.empty(max(cap, 1)); us = np.empty(max(cap, 1)); vs = np.empty(max(cap, 1))
        n = _lib.check(_lib.lib().gwn_ray_tris_hits(
            C.byref(b), _p(O), _p(D), R, float(t_lo), float(t_hi), float(tang_eps),
            float(plane_tol), _p(offs, C.c_int64), _p(ts), _p(tris, C.c_int64), _p(dd),
            _p(us), _p(vs), cap, device), "gwn_ray_tris_hits")
        if n <= cap:
            break
        cap = n
    del keep
    return offs, ts[:n], tris[:n], dd[:n], us[:n], vs[:n]


def bvh_ray_all_hits(bvh, origin, direction, t_lo, t_hi, tang_eps, plane_tol, device: int = 0):
    """All ray hits against a prebuilt BVH; raw arrays ``(ts, tris, dotdn,
    us, vs)`` (_kernels.py:366-381), in the numpy twin's order."""
    _, ts, tris, dd, us, vs = ray_tris_hits_batch(
        bvh, np.asarray(origin, np.float64).reshape(1, 3),
        np.asarray(direction, np.float64).reshape(1, 3), t_lo, t_hi, tang_eps, plane_tol, device)
    return ts, tris, dd, us, vs
