"""Prototype (development aid, not used by the product): the translation
identities behind csrc/gwn_fmm.cu and the Stokes form of the moments in
csrc/gwn_farfield.cu, checked numerically with the solid harmonics of
proto.py.

  M2L  I_n^m(b + x) = sum_{j,k} (-1)^j conj(R_j^k(x)) I_{n+j}^{m+k}(b)
  L2L  R_n^m(x + y) = sum_{a,b} R_a^b(x) R_{n-a}^{m-b}(y)
  D_n^m (area integral over the fan) = -1/(n+1) loop (d x conj(grad R_n^m(d))) . dd
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from proto import irregular, loop_of_patch, moments, omega_exact, omega_mp, regular  # noqa: E402

K = 20
P = 20


def full(T):
    """(n, m >= 0) -> complex, extended to m < 0 by X_n^{-m} = (-1)^m conj(X_n^m)."""
    F = {}
    for (n, m), v in T.items():
        v = v[0] if isinstance(v, tuple) else v
        F[(n, m)] = v
        if m > 0:
            F[(n, -m)] = (-1) ** m * np.conj(v)
    return F


def m2l(D, b):
    Ib = full(irregular(*b, K + P))
    return {(j, k): -(-1) ** j * sum(D[(n, m)] * Ib.get((n + j, m + k), 0)
                                     for n in range(1, K + 1) for m in range(-n, n + 1))
            for j in range(P + 1) for k in range(j + 1)}


def l2p(L, x):
    R = regular(*x, P)
    s = 0.0
    for j in range(P + 1):
        s += (np.conj(R[(j, 0)][0]) * L[(j, 0)]).real
        for k in range(1, j + 1):
            s += 2 * (np.conj(R[(j, k)][0]) * L[(j, k)]).real
    return s


def l2l(L, y):
    R = full(regular(*y, P))
    Lf = full(L)
    return {(a, b): sum(np.conj(R[(j - a, k - b)]) * Lf[(j, k)]
                        for j in range(a, P + 1) for k in range(-j, j + 1)
                        if abs(k - b) <= j - a)
            for a in range(P + 1) for b in range(a + 1)}


def stokes_moments(V, Kt):
    g = V.mean(0)
    A = V - g
    B = np.roll(A, -1, axis=0)
    xg, wg = np.polynomial.legendre.leggauss(Kt // 2 + 1)
    xg, wg = 0.5 * (xg + 1), 0.5 * wg
    D = {}
    for s, w in zip(xg, wg):
        Q = (1 - s) * A + s * B
        R = regular(Q[:, 0], Q[:, 1], Q[:, 2], Kt)
        for (n, m), (_, dx, dy, dz) in R.items():
            if n == 0:
                continue
            G = np.stack([np.conj(dx), np.conj(dy), np.conj(dz)], 1)
            v = -w / (n + 1) * np.einsum("ij,ij->i", np.cross(Q.astype(complex), G), B - A).sum()
            D[(n, m)] = D.get((n, m), 0) + v
    return D


if __name__ == "__main__":
    V = loop_of_patch()
    # proto.moments integrates the fan with 7x7 Gauss points: exact to order 12
    _, _, _, D12 = moments(V, 12)
    Ds = stokes_moments(V, 12)
    print("Stokes vs area moments (order 12), max rel err:",
          max(abs(Ds[k] - D12[k]) / abs(D12[k]) for k in Ds if abs(D12[k]) > 0))
    g, rho, aabs, Dd = moments(V, K)
    D = full(Dd)
    rng = np.random.default_rng(2)
    for dist in (4, 6):
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        z = g + dist * rho * u
        L = m2l(D, z - g)
        y = rng.normal(size=3) * 0.2 * rho
        Lc = l2l(L, y)
        x = rng.normal(size=3)
        x *= 0.3 * rho / np.linalg.norm(x)
        p = z + y + x
        print(f"box at {dist} rho: local {l2p(Lc, x):+.15f} multipole {omega_mp(p, g, Dd, K):+.15f} "
              f"exact {omega_exact(p, V, g):+.15f}")
