"""Seeded synthetic scenes for BASELINE.json configs 1-5.

There is no public dataset for this path: BASELINE.json's five configs are
synthetic bicubic-patch scenes, restated here from SURVEY.md §8(d) with the
open questions of SURVEY Appendix B decided as DESIGN.md §Inputs records
(4x4x2 box lattice for the 64-patch closed surfaces, C5 centres U[-5,5]^3,
C3 "inflated by 50%" = extent x1.5 about the centre).

Control-point layout everywhere: ``ctrl[p, i, j, :]`` with ``i`` the u index
and ``j`` the v index, f(u,v) = sum_ij B_i(u) B_j(v) ctrl[i, j]; the patch
normal is f_u x f_v and the boundary loop runs counter-clockwise in (u,v)
(reference ``CoonsPatch.domain_edges``, pkg/src/gwn/surfaces.py:566-573).

Seeds: ``np.random.default_rng(240804466 + config_index)``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 240804466

#: full query counts per config (BASELINE.json configs[0..4])
FULL_QUERIES = {1: 4096, 2: 1 << 20, 3: 1 << 22, 4: 1 << 24, 5: 1 << 26}


@dataclass
class SceneSpec:
    config: int
    ctrl: np.ndarray            # (P, 4, 4, 3) float64
    queries: np.ndarray         # (Q, 3) float64
    closed: bool                # watertight (integer w expected)
    meta: dict = field(default_factory=dict)

    @property
    def n_patches(self) -> int:
        return int(self.ctrl.shape[0])


# ---------------------------------------------------------------------------
# bicubic evaluation (vectorised; host-side helper, not the hot path)
# ---------------------------------------------------------------------------


def bernstein3(t: np.ndarray) -> np.ndarray:
    t = np.asarray(t, dtype=np.float64)
    s = 1.0 - t
    return np.stack([s * s * s, 3.0 * t * s * s, 3.0 * t * t * s, t * t * t], axis=-1)


def bernstein3_d(t: np.ndarray) -> np.ndarray:
    t = np.asarray(t, dtype=np.float64)
    s = 1.0 - t
    return np.stack([-3.0 * s * s, 3.0 * s * s - 6.0 * t * s, 6.0 * t * s - 3.0 * t * t,
                     3.0 * t * t], axis=-1)


def eval_patches(ctrl: np.ndarray, pid: np.ndarray, u: np.ndarray, v: np.ndarray):
    """Points, f_u, f_v of patches ``pid`` at (u, v) (all arrays length n)."""
    c = ctrl[pid]                       # (n,4,4,3)
    bu, bv = bernstein3(u), bernstein3(v)
    du, dv = bernstein3_d(u), bernstein3_d(v)
    pt = np.einsum("ni,nj,nijk->nk", bu, bv, c)
    fu = np.einsum("ni,nj,nijk->nk", du, bv, c)
    fv = np.einsum("ni,nj,nijk->nk", bu, dv, c)
    return pt, fu, fv


def flip_patch(ctrl_p: np.ndarray) -> np.ndarray:
    """Orientation flip by the u<->v transpose."""
    return np.ascontiguousarray(np.swapaxes(ctrl_p, 0, 1))


# ---------------------------------------------------------------------------
# closed lattice surfaces
# ---------------------------------------------------------------------------

# (normal axis, sign) -> (u axis, v axis) with e_u x e_v = sign * e_normal
_FACE_AXES = {
    (0, +1): (1, 2), (0, -1): (2, 1),
    (1, +1): (2, 0), (1, -1): (0, 2),
    (2, +1): (0, 1), (2, -1): (1, 0),
}


def box_lattice_surface(n_patch: tuple[int, int, int], half: tuple[float, float, float],
                        rng: np.random.Generator, jitter: float,
                        project: str) -> np.ndarray:
    """Closed surface of bicubic patches on the faces of a box lattice.

    ``n_patch[a]`` patches along axis a; every patch has 3 control intervals
    so the lattice has 3*n+1 points per axis.  Surface lattice points are
    projected onto the unit sphere (``project='sphere'``) or onto the
    ellipsoid with semi-axes ``half`` (``'ellipsoid'``), then jittered once
    each so shared edges stay bit-identical.  Orientation is outward.
    """
    npts = [3 * n + 1 for n in n_patch]
    # distinct surface lattice points in a fixed (x, y, z) lexicographic order
    keys = []
    for ix in range(npts[0]):
        for iy in range(npts[1]):
            for iz in range(npts[2]):
                if ix in (0, npts[0] - 1) or iy in (0, npts[1] - 1) or iz in (0, npts[2] - 1):
                    keys.append((ix, iy, iz))
    index = {k: n for n, k in enumerate(keys)}
    kk = np.asarray(keys, dtype=np.float64)
    half_a = np.asarray(half, dtype=np.float64)
    pos = -half_a + kk * (2.0 * half_a / (np.asarray(npts) - 1))
    if project == "sphere":
        pos = pos / np.linalg.norm(pos, axis=1, keepdims=True)
    elif project == "ellipsoid":
        r = np.linalg.norm(pos / half_a, axis=1, keepdims=True)
        pos = pos / r
    pos = pos + rng.normal(0.0, jitter, size=pos.shape)

    patches = []
    for axis in range(3):
        for sign in (-1, +1):
            ua, va = _FACE_AXES[(axis, sign)]
            fixed = 0 if sign < 0 else npts[axis] - 1
            for pu in range(n_patch[ua]):
                for pv in range(n_patch[va]):
                    c = np.empty((4, 4, 3))
                    for i in range(4):
                        for j in range(4):
                            idx = [0, 0, 0]
                            idx[axis] = fixed
                            idx[ua] = 3 * pu + i
                            idx[va] = 3 * pv + j
                            c[i, j] = pos[index[tuple(idx)]]
                    patches.append(c)
    return np.asarray(patches)


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform SO(3) sample (QR of a Gaussian matrix, sign-fixed)."""
    a = rng.normal(size=(3, 3))
    q, r = np.linalg.qr(a)
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


# ---------------------------------------------------------------------------
# configs
# ---------------------------------------------------------------------------


def config1(n_queries: int | None = None) -> SceneSpec:
    rng = np.random.default_rng(SEED_BASE + 1)
    ctrl = np.empty((1, 4, 4, 3))
    z = rng.normal(0.0, 0.2, size=(4, 4))
    for i in range(4):
        for j in range(4):
            ctrl[0, i, j] = (i / 3.0, j / 3.0, z[i, j])
    q = n_queries or FULL_QUERIES[1]
    queries = rng.uniform(-0.5, 1.5, size=(q, 3))
    return SceneSpec(1, ctrl, queries, closed=False)


def config2(n_queries: int | None = None) -> SceneSpec:
    rng = np.random.default_rng(SEED_BASE + 2)
    ctrl = box_lattice_surface((1, 1, 1), (1.0, 1.0, 1.0), rng, 0.05, "sphere")
    q = n_queries or FULL_QUERIES[2]
    queries = rng.uniform(-1.5, 1.5, size=(q, 3))
    return SceneSpec(2, ctrl, queries, closed=True)


def config3(n_queries: int | None = None) -> SceneSpec:
    rng = np.random.default_rng(SEED_BASE + 3)
    a = rng.uniform(-np.pi, np.pi, 4)
    b = rng.uniform(-np.pi, np.pi, 4)
    phi = rng.uniform(0.0, 2.0 * np.pi, 4)
    g = np.arange(25) / 6.0
    X, Y = np.meshgrid(g, g, indexing="ij")
    Z = sum(0.3 * np.sin(a[k] * X + b[k] * Y + phi[k]) for k in range(4))
    Z = Z + rng.normal(0.0, 0.02, size=Z.shape)
    lat = np.stack([X, Y, Z], axis=-1)
    ctrl = np.empty((64, 4, 4, 3))
    for pi in range(8):
        for pj in range(8):
            ctrl[pi * 8 + pj] = lat[3 * pi:3 * pi + 4, 3 * pj:3 * pj + 4]
    q = n_queries or FULL_QUERIES[3]
    n_near = q // 10
    n_far = q - n_near
    lo, hi = ctrl.reshape(-1, 3).min(0), ctrl.reshape(-1, 3).max(0)
    cen, ext = 0.5 * (lo + hi), (hi - lo) * 1.5
    far = cen + (rng.uniform(size=(n_far, 3)) - 0.5) * ext
    pid = rng.integers(0, 64, n_near)
    uu = rng.uniform(size=n_near)
    vv = rng.uniform(size=n_near)
    s = rng.uniform(-1e-3, 1e-3, n_near)
    pt, fu, fv = eval_patches(ctrl, pid, uu, vv)
    nrm = np.cross(fu, fv)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    near = pt + s[:, None] * nrm
    queries = np.concatenate([far, near])
    meta = {"a": a.tolist(), "b": b.tolist(), "phi": phi.tolist(), "n_near": int(n_near)}
    return SceneSpec(3, ctrl, queries, closed=False, meta=meta)


def _deformed_closed_surfaces(rng, n_surf: int, centre_box: float) -> np.ndarray:
    out = []
    for _ in range(n_surf):
        surf = box_lattice_surface((4, 4, 2), (1.0, 1.0, 0.5), rng, 0.05, "ellipsoid")
        rot = random_rotation(rng)
        scale = rng.uniform(0.5, 1.5)
        centre = rng.uniform(-centre_box, centre_box, 3)
        out.append(surf @ rot.T * scale + centre)
    return np.concatenate(out)


def config4(n_queries: int | None = None) -> SceneSpec:
    rng = np.random.default_rng(SEED_BASE + 4)
    ctrl = _deformed_closed_surfaces(rng, 16, 2.0)
    q = n_queries or FULL_QUERIES[4]
    queries = rng.uniform(-3.0, 3.0, size=(q, 3))
    return SceneSpec(4, ctrl, queries, closed=True)


def config5(n_queries: int | None = None) -> SceneSpec:
    rng = np.random.default_rng(SEED_BASE + 5)
    ctrl = _deformed_closed_surfaces(rng, 256, 5.0)
    n = ctrl.shape[0]
    n_del = int(0.05 * n)
    keep = np.sort(rng.permutation(n)[n_del:])
    ctrl = ctrl[keep]
    n_dup = int(0.02 * ctrl.shape[0])
    dup = np.sort(rng.permutation(ctrl.shape[0])[:n_dup])
    flipped = np.asarray([flip_patch(ctrl[k]) for k in dup])
    ctrl = np.concatenate([ctrl, flipped])
    lo, hi = ctrl.reshape(-1, 3).min(0), ctrl.reshape(-1, 3).max(0)
    q = n_queries or FULL_QUERIES[5]
    queries = lo + rng.uniform(size=(q, 3)) * (hi - lo)
    meta = {"deleted": n_del, "duplicated_flipped": n_dup, "centre_box": 5.0}
    return SceneSpec(5, ctrl, queries, closed=False, meta=meta)


def unit_cube(lo=(0.0, 0.0, 0.0), size: float = 1.0) -> np.ndarray:
    """An axis-aligned cube as 6 flat bicubic patches, outward (f_u x f_v)
    orientation -- the SPEC examples' watertight cube."""
    faces = [  # (corner, a, b) with a x b outward
        ((0, 0, 0), (0, 0, 1), (0, 1, 0)), ((1, 0, 0), (0, 1, 0), (0, 0, 1)),
        ((0, 0, 0), (1, 0, 0), (0, 0, 1)), ((0, 1, 0), (0, 0, 1), (1, 0, 0)),
        ((0, 0, 0), (0, 1, 0), (1, 0, 0)), ((0, 0, 1), (1, 0, 0), (0, 1, 0)),
    ]
    lo = np.asarray(lo, np.float64)
    ctrl = np.empty((6, 4, 4, 3))
    for k, (c, a, b) in enumerate(faces):
        c, a, b = (np.asarray(x, np.float64) for x in (c, a, b))
        for i in range(4):
            for j in range(4):
                ctrl[k, i, j] = lo + size * (c + (i / 3.0) * a + (j / 3.0) * b)
    return ctrl


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(config: int, n_queries: int | None = None) -> SceneSpec:
    return CONFIGS[config](n_queries)
