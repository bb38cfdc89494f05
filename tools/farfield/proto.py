"""Prototype (development aid): solid-harmonic far field of a closed polyline's
solid angle, validated against the exact fan sum.  Not used by the product."""
import numpy as np
from math import factorial

K = 10

def regular(x, y, z, K):
    """R[n][m] (0<=m<=n<=K) complex and gradients (value, dx, dy, dz) by recurrence
    with dual numbers: R_0^0 = 1, R_m^m = -(x+iy)/(2m) R_{m-1}^{m-1},
    R_n^m = ((2n-1) z R_{n-1}^m - r^2 R_{n-2}^m) / ((n+m)(n-m))."""
    sh = np.shape(x)
    one = np.ones(sh, complex); zero = np.zeros(sh, complex)
    r2 = x * x + y * y + z * z
    w = x + 1j * y
    R = {}
    R[(0, 0)] = (one, zero, zero, zero)
    for m in range(1, K + 1):
        v, dx, dy, dz = R[(m - 1, m - 1)]
        c = -1.0 / (2 * m)
        R[(m, m)] = (c * w * v, c * (v + w * dx), c * (1j * v + w * dy), c * w * dz)
    for m in range(0, K + 1):
        for n in range(m + 1, K + 1):
            a = R[(n - 1, m)]
            b = R.get((n - 2, m), (zero, zero, zero, zero))
            den = (n + m) * (n - m)
            v = ((2 * n - 1) * z * a[0] - r2 * b[0]) / den
            dx = ((2 * n - 1) * z * a[1] - (2 * x * b[0] + r2 * b[1])) / den
            dy = ((2 * n - 1) * z * a[2] - (2 * y * b[0] + r2 * b[2])) / den
            dz = ((2 * n - 1) * (a[0] + z * a[3]) - (2 * z * b[0] + r2 * b[3])) / den
            R[(n, m)] = (v, dx, dy, dz)
    return R

def irregular(x, y, z, K):
    """I_0^0 = 1/r, I_m^m = -(2m-1)(x+iy)/r^2 I_{m-1}^{m-1},
    I_n^m = ((2n-1) z I_{n-1}^m - ((n-1)^2 - m^2) I_{n-2}^m) / r^2."""
    r2 = x * x + y * y + z * z
    w = x + 1j * y
    I = {(0, 0): 1 / np.sqrt(r2) + 0j}
    for m in range(1, K + 1):
        I[(m, m)] = -(2 * m - 1) * w / r2 * I[(m - 1, m - 1)]
    for m in range(0, K + 1):
        for n in range(m + 1, K + 1):
            b = I.get((n - 2, m), 0)
            I[(n, m)] = ((2 * n - 1) * z * I[(n - 1, m)] - ((n - 1) ** 2 - m * m) * b) / r2
    return I

def addition_check():
    rng = np.random.default_rng(1)
    q = rng.normal(size=3) * 0.1
    p = rng.normal(size=3) * 2
    R = regular(*q, 25); I = irregular(*p, 25)
    s = 0
    for n in range(26):
        for m in range(0, n + 1):
            t = np.conj(R[(n, m)][0]) * I[(n, m)]
            s += t if m == 0 else 2 * t.real
    print("addition theorem:", s.real, 1 / np.linalg.norm(p - q))


def loop_of_patch(seed=3):
    from paper_2408_04466_b200 import scenes
    from paper_2408_04466_b200.surfaces import BicubicPatch
    s = scenes.make(5, 16)
    P = BicubicPatch(s.ctrl[seed])
    L = P.boundary_loops(200)[0]
    return np.asarray(L.points if hasattr(L, "points") else L.vertices, float)


def moments(V, K):
    g = V.mean(0)
    A = V - g
    B = np.roll(A, -1, axis=0)
    nA = np.cross(A, B)                      # (a x b): n dA = nA ds dt
    xg, wg = np.polynomial.legendre.leggauss(7)
    xg = 0.5 * (xg + 1); wg = 0.5 * wg
    D = {}
    for iu, (u, wu) in enumerate(zip(xg, wg)):
        for iv, (v, wv) in enumerate(zip(xg, wg)):
            s, t, jac = u, (1 - u) * v, (1 - u)
            Q = s * A + t * B                 # (T,3) quadrature points (delta)
            R = regular(Q[:, 0], Q[:, 1], Q[:, 2], K)
            for key, (val, dx, dy, dz) in R.items():
                f = (nA[:, 0] * np.conj(dx) + nA[:, 1] * np.conj(dy) + nA[:, 2] * np.conj(dz))
                D[key] = D.get(key, 0) + wu * wv * jac * f.sum()
    rho = np.linalg.norm(V - g, axis=1).max()
    aabs = 0.5 * np.linalg.norm(nA, axis=1).sum()
    return g, rho, aabs, D


def omega_mp(p, g, D, K):
    d = p - g
    I = irregular(d[0], d[1], d[2], K)
    s = 0.0
    for n in range(1, K + 1):
        s += (D[(n, 0)] * I[(n, 0)]).real
        for m in range(1, n + 1):
            s += 2 * (D[(n, m)] * I[(n, m)]).real
    return -s


def omega_exact(p, V, g):
    a = g - p
    b = V - p
    c = np.roll(V, -1, axis=0) - p
    la, lb, lc = np.linalg.norm(a), np.linalg.norm(b, axis=1), np.linalg.norm(c, axis=1)
    num = np.einsum('j,ij->i', a, np.cross(b, c))
    den = la * lb * lc + (b @ a) * lc + (c @ a) * lb + np.einsum('ij,ij->i', b, c) * la
    return (2 * np.arctan2(num, den)).sum()


if __name__ == "__main__":
    addition_check()
    V = loop_of_patch()
    g, rho, aabs, D = moments(V, K)
    print("loop", V.shape, "rho", rho, "A_abs", aabs)
    rng = np.random.default_rng(0)
    for Rr in (2, 3, 5, 10, 20):
        errs = []
        for _ in range(20):
            u = rng.normal(size=3); u /= np.linalg.norm(u)
            p = g + Rr * rho * u
            errs.append(abs(omega_mp(p, g, D, K) - omega_exact(p, V, g)))
        bound = aabs * (K + 2) * rho ** (K + 1) / ((Rr - 1) * rho) ** (K + 3)
        print(f"R/rho {Rr:3d}: max err {max(errs):.2e}  bound {bound:.2e}  |omega| ~ {abs(omega_exact(p, V, g)):.2e}")


def k4_fan(p, V, d):
    """K4's per-loop angle sum: sum 2 atan2(c.(a^ x b^), 1 + a^.b^ + b^.c + c.a^), c = -d."""
    c = -d
    A = V - p; A /= np.linalg.norm(A, axis=1)[:, None]
    B = np.roll(A, -1, axis=0)
    num = np.cross(A, B) @ c
    den = 1 + np.einsum('ij,ij->i', A, B) + B @ c + A @ c
    return (2 * np.arctan2(num, den)).sum()


def sign_check():
    V = loop_of_patch()
    g = V.mean(0)
    rng = np.random.default_rng(5)
    for _ in range(6):
        u = rng.normal(size=3); u /= np.linalg.norm(u)
        p = g + 4 * u
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        r = g - p
        line = np.sqrt(max(r @ r - (r @ d) ** 2, 0))
        print(f"line dist {line:.3f}  k4 {k4_fan(p, V, d):+.12f}  exact {omega_exact(p, V, g):+.12f}")


def bound_check():
    """The truncation bounds of gwn_farfield.cuh against measured errors."""
    V = loop_of_patch()
    for Kt in (6, 8, 10):
        g, rho, aabs, D = moments(V, Kt)
        rng = np.random.default_rng(1)
        for Rr in (1.5, 2, 3, 5, 10):
            errs = []
            for _ in range(40):
                u = rng.normal(size=3); u /= np.linalg.norm(u)
                p = g + Rr * rho * u
                errs.append(abs(omega_mp(p, g, D, Kt) - omega_exact(p, V, g)))
            R = Rr * rho
            tay = aabs * (Kt + 1) * rho ** Kt / (R - rho) ** (Kt + 2)
            leg = 2 ** 0.5 * aabs * (Kt + 1) * (rho / R) ** Kt / (R - rho) ** 2
            print(f"K {Kt} R/rho {Rr}: max err {max(errs):.2e}  bound {min(tay, leg):.2e}  ok {max(errs) <= min(tay, leg)}")
