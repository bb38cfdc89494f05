"""GPU: the rest of the kernel dispatch layer (solid angles, ray/mesh all
hits) through libgwn_b200.so against the reference's own
outputs (tests/golden/mesh.npz) and the CPU oracle (oracle/mesh_oracle.py).

Tolerances: solid-angle totals 1e-11 absolute (one complex product per
query instead of per-triangle atan2 sums), hits and crossing points 1e-12;
indices, flags and orders exact.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_04466_b200 import _kernels as K, scenes  # noqa: E402
from paper_2408_04466_b200.mesh import build_bvh, intersect_ray_mesh, mesh_winding_numbers  # noqa: E402
from paper_2408_04466_b200.geometry import Ray  # noqa: E402
from oracle import mesh_oracle as MO  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "mesh.npz")
SA_TOL = 1e-11


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def tess(ctrl, n):
    g_ = np.linspace(0.0, 1.0, n + 1)
    s = 1.0 - g_
    B = np.stack([s ** 3, 3 * g_ * s * s, 3 * g_ * g_ * s, g_ ** 3], axis=1)
    Vs, Ts, base = [], [], 0
    for P in np.asarray(ctrl).reshape(-1, 4, 4, 3):
        X = np.einsum("ui,vj,ijk->uvk", B, B, P).reshape(-1, 3)
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        a, b = (i * (n + 1) + j).ravel() + base, ((i + 1) * (n + 1) + j).ravel() + base
        Ts.append(np.stack([np.stack([a, b, b + 1], 1), np.stack([a, b + 1, a + 1], 1)], 1)
                  .reshape(-1, 3))
        Vs.append(X)
        base += len(X)
    return np.concatenate(Vs), np.concatenate(Ts).astype(np.int64)


@pytest.mark.parametrize("name", ["closed", "open"])
def test_solid_angle_vs_reference(g, name):
    out, on = K.solid_angle_many(g[f"sa_{name}_V"], g[f"sa_{name}_T"], g[f"sa_{name}_P"])
    assert np.array_equal(on, g[f"sa_{name}_on"].astype(bool))
    assert np.abs(out - g[f"sa_{name}_out"]).max() < SA_TOL
    t, f = K.solid_angle_sum(g[f"sa_{name}_V"], g[f"sa_{name}_T"], g[f"sa_{name}_P"][3])
    assert abs(t - g[f"sa_{name}_out"][3]) < SA_TOL and f == bool(g[f"sa_{name}_on"][3])


def test_solid_angle_large_vs_oracle_and_closed_integers():
    V, T = tess(scenes.config4(8).ctrl[:128], 10)      # 2 closed surfaces, 25.6K triangles
    rng = np.random.default_rng(11)
    P = rng.uniform(-3, 3, (4096, 3))
    out, on = K.solid_angle_many(V, T, P)
    sub = rng.choice(len(P), 96, replace=False)
    ref, ron = MO.solid_angle_many(V, T, P[sub])
    assert np.array_equal(on[sub], ron)
    assert np.abs(out[sub] - ref).max() < 1e-10
    w, won = mesh_winding_numbers(V, T, P)
    # closed (watertight up to the seam round-off): integers away from the surface
    assert np.abs(w - np.round(w)).max() < 1e-3
    assert not won.any()


def test_solid_angle_edge_cases():
    V = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    T = np.array([[0, 1, 2]])
    out, on = K.solid_angle_many(V, T, np.zeros((0, 3)))
    assert out.shape == (0,)
    out, on = K.solid_angle_many(V, np.zeros((0, 3), np.int64), np.ones((3, 3)))
    assert np.all(out == 0) and not on.any()
    # on a vertex, on the face, just above the face
    out, on = K.solid_angle_many(V, T, [[0, 0, 0], [0.2, 0.2, 0], [0.2, 0.2, 1e-3]])
    assert on.tolist() == [True, True, False]
    assert abs(out[2] - MO.solid_angle_sum(V, T, [0.2, 0.2, 1e-3])[0]) < 1e-13
    with pytest.raises(Exception):
        K.solid_angle_many(V, np.array([[0, 1, 7]]), np.ones((1, 3)))


@pytest.mark.parametrize("name", ["sphere", "flat"])
def test_ray_hits_vs_reference(g, name):
    bvh = build_bvh(g[f"hit_{name}_V"], g[f"hit_{name}_T"])
    offs, H = g[f"hit_{name}_offs"], g[f"hit_{name}_hits"]
    tol = float(g[f"hit_{name}_plane_tol"])
    O, D = g[f"hit_{name}_O"], g[f"hit_{name}_D"]
    goffs, ts, tris, dd, us, vs = K.ray_tris_hits_batch(bvh, O, D, 0.0, np.inf, 1e-12, tol)
    assert np.array_equal(goffs, offs)
    mine = np.stack([ts, tris.astype(np.float64), dd, us, vs], axis=1)
    assert np.array_equal(tris, H[:, 1].astype(np.int64))
    assert np.abs(mine - H).max(initial=0.0) <= 1e-12 * (1 + np.abs(H).max(initial=0.0))
    # the per-ray dispatch-layer call (_kernels.py:366)
    r = 5
    t1, f1, d1, u1, v1 = K.bvh_ray_all_hits(bvh, O[r], D[r], 0.0, np.inf, 1e-12, tol)
    assert np.array_equal(f1, H[offs[r]:offs[r + 1], 1].astype(np.int64))


def test_ray_hits_large_vs_oracle_and_records():
    V, T = tess(scenes.config4(8).ctrl[:64], 12)
    bvh = build_bvh(V, T)
    rng = np.random.default_rng(3)
    O = rng.uniform(-3, 3, (2000, 3))
    D = rng.normal(size=(2000, 3))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    offs, ts, tris, dd, us, vs = K.ray_tris_hits_batch(bvh, O, D, 0.0, np.inf, 1e-12, 1e-9)
    arrs = MO.bvh_arrays(V, T)
    for r in rng.choice(2000, 60, replace=False):
        ref = MO.ray_tris_hits(*arrs, O[r], D[r], 0.0, np.inf, 1e-12, 1e-9)
        a, b = offs[r], offs[r + 1]
        assert np.array_equal(tris[a:b], ref[:, 1].astype(np.int64))
        assert np.abs(ts[a:b] - ref[:, 0]).max(initial=0.0) < 1e-12
    # closed surface: hit signs along a ray alternate to a net 0 or +-1 count
    recs = intersect_ray_mesh(V, T, Ray(np.array([-5.0, 0.1, 0.2]), np.array([1.0, 0, 0])),
                              bvh=bvh)
    assert all(recs[k].t <= recs[k + 1].t for k in range(len(recs) - 1))
    empty = K.ray_tris_hits_batch(bvh, np.zeros((0, 3)), np.zeros((0, 3)), 0.0, np.inf, 1e-12,
                                  1e-9)
    assert empty[0].tolist() == [0] and len(empty[1]) == 0
