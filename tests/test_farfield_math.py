"""CPU checks of the far-field math behind K4's expansion (DESIGN §9 f4,
csrc/gwn_farfield.cuh): the solid-harmonic recurrences satisfy the addition
theorem, the double-layer multipole of a closed boundary loop matches its exact
solid angle, the truncation bound holds, and K4's fan sum equals the solid
angle when the ray line misses the loop's sphere.  The numpy restatement lives
in tools/farfield/proto.py (the same recurrences the kernels use)."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tools", "farfield"))
proto = pytest.importorskip("proto")


def test_addition_theorem():
    rng = np.random.default_rng(7)
    for _ in range(5):
        q = rng.normal(size=3) * 0.2
        p = rng.normal(size=3)
        p *= 2.0 / np.linalg.norm(p)
        R = proto.regular(*q, 30)
        I = proto.irregular(*p, 30)
        s = 0.0
        for n in range(31):
            for m in range(n + 1):
                t = np.conj(R[(n, m)][0]) * I[(n, m)]
                s += t.real if m == 0 else 2 * t.real
        assert abs(s - 1 / np.linalg.norm(p - q)) < 1e-15


def test_multipole_matches_exact_solid_angle_within_bound():
    V = proto.loop_of_patch()
    K = 8
    g, rho, aabs, D = proto.moments(V, K)
    rng = np.random.default_rng(3)
    for Rr in (3.0, 6.0, 12.0):
        R = Rr * rho
        taylor = aabs * (K + 1) * rho ** K / (R - rho) ** (K + 2)
        legendre = 2 ** 0.5 * aabs * (K + 1) * (rho / R) ** K / (R - rho) ** 2
        bound = min(taylor, legendre)
        for _ in range(8):
            u = rng.normal(size=3)
            p = g + R * u / np.linalg.norm(u)
            err = abs(proto.omega_mp(p, g, D, K) - proto.omega_exact(p, V, g))
            assert err <= bound, (Rr, err, bound)


def test_fan_sum_equals_solid_angle_when_line_misses_sphere():
    V = proto.loop_of_patch()
    g = V.mean(0)
    rho = np.linalg.norm(V - g, axis=1).max()
    rng = np.random.default_rng(5)
    checked = 0
    while checked < 10:
        u = rng.normal(size=3)
        p = g + 4.0 * u / np.linalg.norm(u)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        r = g - p
        if r @ r - (r @ d) ** 2 <= (1.01 * rho) ** 2:
            continue
        # proto.k4_fan is K4's fan formula in full angles (the kernel stores halves)
        assert abs(proto.k4_fan(p, V, d) - proto.omega_exact(p, V, g)) < 1e-13
        checked += 1


def test_irregular_harmonic_bound_and_tail_bound():
    """The a-posteriori order thresholds (gwn_farfield.cu): |I_n^m(x)| <=
    sqrt((n-m)! (n+m)!) / |x|^(n+1), so truncating the expansion at order p < K
    changes it by at most sum_{n=p+1..K} T_n / R^(n+1) with
    T_n = |D_n^0| n! + 2 sum_{m>=1} |D_n^m| sqrt((n-m)! (n+m)!)."""
    from math import factorial, sqrt
    rng = np.random.default_rng(11)
    K = 24
    worst = 0.0
    for _ in range(40):
        u = rng.normal(size=3)
        r = rng.uniform(0.5, 3.0)
        p = r * u / np.linalg.norm(u)
        I = proto.irregular(p[0], p[1], p[2], K)
        for n in range(K + 1):
            for m in range(n + 1):
                b = sqrt(factorial(n - m) * factorial(n + m)) / r ** (n + 1)
                worst = max(worst, abs(I[(n, m)]) / b)
    assert worst <= 1.0 + 1e-12
    # the tail bound against the actual difference of two truncations
    V = proto.loop_of_patch()
    g, rho, aabs, D = proto.moments(V, K)
    T = np.zeros(K + 1)
    for n in range(1, K + 1):
        for m in range(n + 1):
            T[n] += (2.0 if m else 1.0) * abs(D[(n, m)]) * sqrt(factorial(n - m) * factorial(n + m))
    for Rr in (1.5, 2.5, 5.0):
        R = Rr * rho
        for pl in (8, 12, 16):
            tail = sum(T[n] / R ** (n + 1) for n in range(pl + 1, K + 1))
            for _ in range(6):
                u = rng.normal(size=3)
                p = g + R * u / np.linalg.norm(u)
                diff = abs(proto.omega_mp(p, g, D, K) - proto.omega_mp(p, g, D, pl))
                assert diff <= tail * (1 + 1e-9) + 1e-18, (Rr, pl, diff, tail)
