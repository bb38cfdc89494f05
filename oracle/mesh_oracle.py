"""CPU oracle for the rest of the kernel dispatch layer -- TEST INFRASTRUCTURE
ONLY (imported by tests/ as the checker; never by the product path).

A numpy restatement of the reference's numpy twins, which are the correct
versions (the numba kernels share the broken _cross helper,
pkg/src/gwn/_kernels.py:45):
  * solid_angle_sum       _kernels.py:422-440 (_solid_angle_numpy), :443-451
  * ray_tris_hits         _kernels.py:312-363 (_ray_tris_hits_numpy), the
                          brute-force twin of bvh_ray_all_hits :366-381

Parity pinned by tests/test_oracle_golden.py against tests/golden/mesh.npz,
which tests/golden/make_golden_mesh.py generates by running the reference.
"""

from __future__ import annotations

import math

import numpy as np


def solid_angle_sum(V, T, p, guard=1e-12):
    """(sum_f 2 atan2(num, den), on_surface) -- _kernels.py:422-440."""
    V = np.asarray(V, np.float64)
    T = np.asarray(T, np.int64)
    p = np.asarray(p, np.float64)
    a, b, c = V[T[:, 0]] - p, V[T[:, 1]] - p, V[T[:, 2]] - p
    la = np.sqrt(np.einsum("ij,ij->i", a, a))
    lb = np.sqrt(np.einsum("ij,ij->i", b, b))
    lc = np.sqrt(np.einsum("ij,ij->i", c, c))
    num = np.einsum("ij,ij->i", a, np.cross(b, c))
    den = (la * lb * lc + np.einsum("ij,ij->i", a, b) * lc
           + np.einsum("ij,ij->i", b, c) * la + np.einsum("ij,ij->i", c, a) * lb)
    # on a vertex, or coplanar with a triangle inside its rim (:434-435)
    near = (la < guard) | (lb < guard) | (lc < guard)
    near |= (np.abs(num) < guard * la * lb * lc) & (den <= 0.0)
    om = 2.0 * np.arctan2(num, den)
    return float(np.sum(om[~near])), bool(np.any(near))


def solid_angle_many(V, T, P, guard=1e-12):
    P = np.asarray(P, np.float64).reshape(-1, 3)
    out = np.empty(len(P))
    on = np.zeros(len(P), bool)
    for k, p in enumerate(P):
        out[k], on[k] = solid_angle_sum(V, T, p, guard)
    return out, on


def ray_tris_hits(V0, E1, E2, NN, NH, C, R2, origin, direction, t_lo, t_hi, tang_eps,
                  plane_tol):
    """Brute-force all hits (t, tri, dotdn, u, v) -- _kernels.py:312-363:
    regular hits in triangle order, then parallel tangent contacts."""
    o = np.asarray(origin, np.float64)
    d = np.asarray(direction, np.float64)
    h = np.cross(np.broadcast_to(d, E2.shape), E2)
    a = np.einsum("ij,ij->i", E1, h)
    s = o - V0
    par = np.abs(a) <= tang_eps * NN
    hits = []
    reg = ~par
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = np.where(reg, 1.0 / np.where(reg, a, 1.0), 0.0)
        u = inv * np.einsum("ij,ij->i", s, h)
        q = np.cross(s, E1)
        v = inv * (q @ d)
        t = inv * np.einsum("ij,ij->i", E2, q)
    ok = reg & (u >= -1e-12) & (u <= 1.0 + 1e-12) & (v >= -1e-12) & (u + v <= 1.0 + 1e-12) \
        & (t >= t_lo) & (t <= t_hi)
    for f in np.nonzero(ok)[0]:
        hits.append((t[f], f, -a[f] / NN[f], u[f], v[f]))
    pidx = np.nonzero(par)[0]
    if pidx.size:
        pdist = np.abs(np.einsum("ij,ij->i", s[pidx], NH[pidx]))
        tc = C[pidx] - o
        tca = tc @ d
        d2 = np.einsum("ij,ij->i", tc, tc) - tca * tca
        good = (pdist <= plane_tol) & (d2 <= R2[pidx]) & (tca >= t_lo) & (tca <= t_hi)
        for k in np.nonzero(good)[0]:
            hits.append((tca[k], pidx[k], 0.0, 1.0 / 3.0, 1.0 / 3.0))
    return np.asarray(hits, np.float64).reshape(-1, 5)


def bvh_arrays(V, T):
    """Per-triangle Moller-Trumbore data of surfaces.py:147-163 (build_bvh)."""
    V = np.asarray(V, np.float64)
    T = np.asarray(T, np.int64)
    p0, p1, p2 = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    cent = (p0 + p1 + p2) / 3.0
    e1, e2 = p1 - p0, p2 - p0
    n = np.cross(e1, e2)
    nn = np.linalg.norm(n, axis=1)
    nh = n / np.where(nn > 0, nn, 1.0)[:, None]
    r2 = np.maximum(np.maximum(np.einsum("ij,ij->i", p0 - cent, p0 - cent),
                               np.einsum("ij,ij->i", p1 - cent, p1 - cent)),
                    np.einsum("ij,ij->i", p2 - cent, p2 - cent))
    return p0, e1, e2, nn, nh, cent, r2
