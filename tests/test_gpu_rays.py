"""Ray reuse: gwn_eval_rays,
winding_numbers_along_ray, slice and voxelize against the per-point engine
(itself parity-tested against the oracle) and the oracle directly.

Bars from SPEC.md:381-407: ray reuse equals per-point evaluation within
1e-9; slice casts min(W, H) rays, voxelize N^2.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_04466_b200 as G  # noqa: E402
from paper_2408_04466_b200 import scenes  # noqa: E402
from oracle import oracle as O  # noqa: E402

TOL = 1e-9  # SPEC.md:385 "results equal pointwise winding_number within 1e-9"


def unit_cube() -> np.ndarray:
    return scenes.unit_cube()


def _random_rays(rng, lo, hi, R, K):
    org = lo + rng.uniform(size=(R, 3)) * (hi - lo)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    span = np.linalg.norm(hi - lo)
    ts = np.sort(rng.uniform(-0.5 * span, 0.5 * span, size=(R, K)), axis=1).ravel()
    offs = np.arange(R + 1, dtype=np.int64) * K
    pts = np.repeat(org, K, axis=0) + ts[:, None] * d[None, :]
    return org, d, ts, offs, pts


def _cmp(w, st, wp, sp, exact=False):
    m = (st == 0) & (sp == 0)
    assert m.mean() > 0.99, (np.unique(st, return_counts=True), np.unique(sp, return_counts=True))
    if exact:
        assert np.array_equal(w[m], wp[m])
    else:
        assert np.abs(w - wp)[m].max() <= TOL
    return m


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_rays_match_per_point(cfg):
    s = scenes.make(cfg, 16)
    sc = G.Scene(s.ctrl)
    lo, hi = s.ctrl.reshape(-1, 3).min(0), s.ctrl.reshape(-1, 3).max(0)
    rng = np.random.default_rng(100 + cfg)
    org, d, ts, offs, pts = _random_rays(rng, lo, hi, 64, 100)
    w, st, cast = G.winding_numbers_rays(sc, org, d, ts, offs, return_rays=True)
    assert cast == 64
    wp, sp = G.winding_numbers(sc, pts)
    _cmp(w, st, wp, sp, exact=s.closed)


def test_along_ray_matches_oracle():
    s = scenes.make(1, 16)
    sc = G.Scene(s.ctrl)
    rng = np.random.default_rng(7)
    o = rng.uniform(-0.5, 1.5, 3)
    d = rng.normal(size=3)
    ts = np.sort(rng.uniform(-2, 2, 100))
    w = np.array(G.winding_numbers_along_ray(sc, G.Ray(o, d / np.linalg.norm(d)), ts))
    assert sc.rays_cast == 1
    pts = o + ts[:, None] * (d / np.linalg.norm(d))
    wo, so, _, _ = O.scene_eval(s.ctrl, pts)
    assert np.abs(w - wo)[so == 0].max() <= TOL
    assert G.winding_numbers_along_ray(sc, G.Ray(o, d), []) == []


def test_spec_ray_examples_cube():
    sc = G.Scene(unit_cube())
    # ray through the cube, ts straddling both walls -> {0, 1, 0}
    w = G.winding_numbers_along_ray(sc, G.Ray(np.array([-1.0, 0.3, 0.6]),
                                              np.array([1.0, 0.0, 0.0])), [0.5, 1.5, 2.5])
    assert w == [0.0, 1.0, 0.0]
    # slice W=3, H=5 -> exactly 3 rays
    img = G.slice(sc, [-0.25, -0.25, 0.5], [1.5, 0, 0], [0, 1.5, 0], 3, 5)
    assert img.shape == (5, 3) and sc.rays_cast == 3
    # slice through the centre -> binary point-in-cube image
    img = G.slice(sc, [-0.25, -0.25, 0.5], [1.5, 0, 0], [0, 1.5, 0], 32, 32)
    assert sc.rays_cast == 32
    c = -0.25 + (np.arange(32) + 0.5) / 32 * 1.5
    inside = ((c[:, None] > 0) & (c[:, None] < 1)) & ((c[None, :] > 0) & (c[None, :] < 1))
    assert np.array_equal(img, inside.astype(np.float64))  # img[j, i]: y=c[j], x=c[i]
    # voxelize [0,1]^3 at N=2 -> 8 occupied; outside the AABB -> 0
    occ, w = G.voxelize(sc, 2, [0, 0, 0], [1, 1, 1])
    assert occ.sum() == 8 and sc.rays_cast == 4
    occ, w = G.voxelize(sc, 4, [2, 2, 2], [3, 3, 3])
    assert occ.sum() == 0 and sc.rays_cast == 16


def test_slice_matches_per_pixel_open_patch():
    s = scenes.make(3, 16)
    sc = G.Scene(s.ctrl)
    o, u, v = np.array([-0.3, -0.2, 0.1]), np.array([4.6, 0.3, 0.0]), np.array([0.2, 4.5, 0.05])
    for W, H in ((32, 32), (40, 17), (9, 50)):
        img = G.slice(sc, o, u, v, W, H)
        assert sc.rays_cast == min(W, H) and img.shape == (H, W)
        jj, ii = np.meshgrid((np.arange(H) + 0.5) / H, (np.arange(W) + 0.5) / W, indexing="ij")
        pts = o + ii.ravel()[:, None] * u + jj.ravel()[:, None] * v
        wp, sp = G.winding_numbers(sc, pts)
        assert np.abs(img.ravel() - wp)[sp == 0].max() <= TOL


@pytest.mark.parametrize("cfg,n", [(4, 48), (5, 24)])
def test_voxelize_matches_per_point(cfg, n):
    s = scenes.make(cfg, 16)
    sc = G.Scene(s.ctrl)
    occ, w = G.voxelize(sc, n)
    assert sc.rays_cast == n * n and w.shape == (n, n, n)
    bb = sc.aabb()
    c = (np.arange(n) + 0.5) / n
    ax = [bb.min_corner[k] + c * (bb.max_corner[k] - bb.min_corner[k]) for k in range(3)]
    X, Y, Z = np.meshgrid(*ax, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    wp, sp = G.winding_numbers(sc, pts)
    if cfg == 4:  # closed: integer-exact away from the surface
        assert np.array_equal(w.ravel()[sp == 0], wp[sp == 0])
    else:
        assert np.abs(w.ravel() - wp)[sp == 0].max() <= TOL
    assert np.array_equal(occ, w >= 0.5)


def test_ragged_and_empty_rays():
    s = scenes.make(3, 16)
    sc = G.Scene(s.ctrl)
    rng = np.random.default_rng(3)
    R = 50
    counts = rng.integers(0, 6, R)
    counts[[0, 7, R - 1]] = 0
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    org = rng.uniform(-0.5, 4.5, size=(R, 3))
    d = np.array([0.3, -0.2, 1.0])
    d /= np.linalg.norm(d)
    ts = np.concatenate([np.sort(rng.uniform(-3, 3, c)) for c in counts])
    w, st = G.winding_numbers_rays(sc, org, d, ts, offs)
    pts = np.repeat(org, counts, axis=0) + ts[:, None] * d
    wp, sp = G.winding_numbers(sc, pts)
    _cmp(w, st, wp, sp)
    # points exactly on the surface clash with a hit -> per-point engine (status 1)
    pid = np.array([5, 20, 40])
    pt, _, _ = scenes.eval_patches(s.ctrl, pid, np.array([0.3, 0.5, 0.7]), np.array([0.6, 0.5, 0.2]))
    org2 = pt - 2.0 * d
    w2, st2 = G.winding_numbers_rays(sc, org2, d, np.full(3, 2.0), np.arange(4, dtype=np.int64))
    assert np.all(st2 == 1)
    with pytest.raises(ValueError):
        G.winding_numbers_rays(sc, org, d, ts[::-1].copy(), offs)
