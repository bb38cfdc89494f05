"""CPU: the mesh oracle (oracle/mesh_oracle.py) pinned against the
reference's own numpy twins (tests/golden/mesh.npz, make_golden_mesh.py),
and the product's BVH builder (its own Morton-order build in the
reference's Bvh array layout) against the layout invariants and the
reference's per-triangle arrays."""

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
    # leaf boxes are the exact bounds of their triangles
    for k in np.nonzero(leaves & (b.node_count > 0))[0]:
        ids = b.tri_order[b.node_start[k]:b.node_start[k] + b.node_count[k]]
        P = V[T[ids]].reshape(-1, 3)
        assert np.array_equal(P.min(axis=0), b.node_min[k])
        assert np.array_equal(P.max(axis=0), b.node_max[k])
    arrs = MO.bvh_arrays(V, T)
    for x, y in zip((b.V0, b.E1, b.E2, b.NN, b.NH, b.C), arrs[:6]):
        assert np.array_equal(x, y)
    # squared circumradius (box widening only): within a few ulp
    assert np.all(np.abs(b.R2 - arrs[6]) <= 4 * np.spacing(arrs[6]))
