"""CPU: the mesh / arc oracle (oracle/mesh_oracle.py) pinned against the
reference's own numpy twins (tests/golden/mesh.npz, make_golden_mesh.py),
and the product's BVH builder against the reference's build_bvh arrays."""

import os

import numpy as np
import pytest

from oracle import mesh_oracle as MO

GOLD = os.path.join(os.path.dirname(__file__), "golden", "mesh.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


@pytest.mark.parametrize("name", ["closed", "open"])
def test_solid_angle_oracle_vs_reference(g, name):
    out, on = MO.solid_angle_many(g[f"sa_{name}_V"], g[f"sa_{name}_T"], g[f"sa_{name}_P"])
    assert np.array_equal(on, g[f"sa_{name}_on"].astype(bool))
    assert np.abs(out - g[f"sa_{name}_out"]).max() < 1e-12
    assert on.sum() >= 8  # the planted on-surface points


@pytest.mark.parametrize("name", ["sphere", "flat"])
def test_ray_hits_oracle_vs_reference(g, name):
    arrs = MO.bvh_arrays(g[f"hit_{name}_V"], g[f"hit_{name}_T"])
    offs, H = g[f"hit_{name}_offs"], g[f"hit_{name}_hits"]
    tol = float(g[f"hit_{name}_plane_tol"])
    for r, (o, d) in enumerate(zip(g[f"hit_{name}_O"], g[f"hit_{name}_D"])):
        mine = MO.ray_tris_hits(*arrs, o, d, 0.0, np.inf, 1e-12, tol)
        ref = H[offs[r]:offs[r + 1]]
        assert mine.shape == ref.shape
        assert np.array_equal(mine[:, 1], ref[:, 1])
        assert np.abs(mine - ref).max(initial=0.0) <= 1e-12 * (1 + np.abs(ref).max(initial=0.0))
    if name == "flat":
        assert np.any(H[:, 2] == 0.0)  # parallel tangent contacts are exercised


@pytest.mark.parametrize("name", ["eight", "star", "patch"])
def test_arc_crossings_oracle_vs_reference(g, name):
    k = lambda s: g[f"arc_{name}_{s}"]  # noqa: E731
    pi, pj, pp, ci, cj = MO.arc_crossings(k("S"), k("E"), k("P"), k("L"), k("prev"), k("next"),
                                          1e-9, 1e-12)
    assert np.array_equal(pi, k("pi")) and np.array_equal(pj, k("pj"))
    assert np.abs(pp - k("pts")).max(initial=0.0) < 1e-14
    assert np.array_equal(ci, k("ci")) and np.array_equal(cj, k("cj"))


def test_build_bvh_matches_reference_layout(g):
    from paper_2408_04466_b200.mesh import build_bvh
    V, T = g["hit_sphere_V"], g["hit_sphere_T"]
    b = build_bvh(V, T)
    # every triangle sits in exactly one leaf, leaves cover tri_order
    leaves = b.node_left < 0
    assert b.node_count[leaves].sum() == len(T)
    assert np.array_equal(np.sort(b.tri_order), np.arange(len(T)))
    assert np.all(b.node_count[leaves] <= 8)
    # children boxes inside their parent's
    inner = np.nonzero(~leaves)[0]
    for c in (b.node_left[inner], b.node_right[inner]):
        assert np.all(b.node_min[c] >= b.node_min[inner] - 1e-15)
        assert np.all(b.node_max[c] <= b.node_max[inner] + 1e-15)
    arrs = MO.bvh_arrays(V, T)
    for x, y in zip((b.V0, b.E1, b.E2, b.NN, b.NH, b.C, b.R2), arrs):
        assert np.array_equal(x, y)
