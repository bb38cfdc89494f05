"""CPU: scene ingestion, patch-type conversions and wire formats
 -- conversions pinned against the
reference's own CoonsPatch / BezierTrianglePatch (tests/golden/mesh.npz)."""

import json
import os

import numpy as np
import pytest

from paper_2408_04466_b200 import cli, formats as F, scenes
from paper_2408_04466_b200.errors import GridMismatch, SceneError
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "mesh.npz")


def bic(net, s, t):
    b = lambda x: np.array([(1 - x) ** 3, 3 * x * (1 - x) ** 2, 3 * x * x * (1 - x), x ** 3])  # noqa
    return np.einsum("i,j,ijk->k", b(s), b(t), net)


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def test_coons_conversion_matches_reference(g):
    net = F.coons_to_bicubic(*g["coons_curves"])
    pts = np.array([bic(net, u, v) for u, v in g["coons_uv"]])
    assert np.abs(pts - g["coons_pts"]).max() < 1e-14
    # u-partial by a central difference of the net (reference partials :536-553)
    h = 1e-6
    du = np.array([(bic(net, u + h, v) - bic(net, u - h, v)) / (2 * h) for u, v in g["coons_uv"]])
    assert np.abs(du - g["coons_du"]).max() < 1e-7
    # boundary: the 4 net edges sampled like patch_boundary (surfaces.py:611-626)
    ec, w = O.net_boundary(net[None])
    mine = np.concatenate([O.sample_edge(e, 20)[:-1] for e in ec])
    ref = g["coons_loop"]
    assert mine.shape == ref.shape
    key = lambda a: a[np.lexsort(np.round(a, 12).T)]  # noqa: E731
    assert np.abs(key(mine) - key(ref)).max() < 1e-13


def test_bezier_triangle_conversion_matches_reference(g):
    C = g["tri_control"]
    net = F.bezier_triangle_to_bicubic(C)
    uv = g["tri_uv"]
    t = uv[:, 1]
    s = np.where(t < 1, uv[:, 0] / np.maximum(1 - t, 1e-300), 0.0)
    pts = np.array([bic(net, a, b) for a, b in zip(s, t)])
    assert np.abs(pts - g["tri_pts"]).max() < 1e-13
    # boundary: 3 live edges + 1 collapsed (dropped), same loop as the reference
    ec, w = O.net_boundary(net[None])
    assert len(ec) == 3
    mine = np.concatenate([O.sample_edge(e, 20)[:-1] for e in ec])
    ref = g["tri_loop"]
    key = lambda a: a[np.lexsort(np.round(a, 12).T)]  # noqa: E731
    assert mine.shape == ref.shape and np.abs(key(mine) - key(ref)).max() < 1e-13
    # orientation: the bicubic normal agrees with the triangle's f_u x f_v
    h = 1e-6
    su, sv = 0.3, 0.4
    n_b = np.cross((bic(net, su + h, sv) - bic(net, su - h, sv)),
                   (bic(net, su, sv + h) - bic(net, su, sv - h)))
    u, v = su * (1 - sv), sv
    fu = F.bezier_triangle_point(C, u + h, v) - F.bezier_triangle_point(C, u - h, v)
    fv = F.bezier_triangle_point(C, u, v + h) - F.bezier_triangle_point(C, u, v - h)
    assert np.dot(n_b, np.cross(fu, fv)) > 0


def test_scene_parsing_and_errors(tmp_path):
    cube = scenes.unit_cube()
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]) + 5
    T = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]])
    F.write_obj(str(tmp_path / "tet.obj"), V, T)
    doc = {"boundary_samples_per_edge": 300, "epsilons": {"dedup": 1e-9},
           "patches": [{"type": "bicubic", "control": cube[0].tolist()},
                       {"type": "coons", "curves": {"c0": cube[1, :, 0].tolist(),
                                                    "c1": cube[1, :, 3].tolist(),
                                                    "d0": cube[1, 0, :].tolist(),
                                                    "d1": cube[1, 3, :].tolist()}},
                       {"type": "bezier_triangle", "control": np.eye(3).tolist() * 3 + [[0, 0, 0]]},
                       {"type": "mesh_obj", "path": "tet.obj"}]}
    (tmp_path / "s.json").write_text(json.dumps(doc))
    spec = F.load_scene(str(tmp_path / "s.json"))
    assert spec.ctrl.shape == (3, 4, 4, 3) and spec.samples_per_edge == 300
    assert np.abs(spec.ctrl[1] - cube[1]).max() < 1e-15   # a flat face is its own Coons patch
    V2, T2 = spec.meshes[0]
    assert np.array_equal(V2, V) and np.array_equal(T2, T)
    bad = [{}, {"patches": [{"type": "nurbs"}]}, {"patches": [{"type": "bem_loop"}]},
           {"patches": [{"type": "bicubic", "control": [[0, 0, 0]]}]},
           {"patches": [{"type": "bezier_triangle", "control": [[0, 0, 0]] * 9}]},
           {"patches": [{"type": "mesh_obj", "path": "missing.obj"}]},
           {"patches": [], "boundary_samples_per_edge": 1}]
    for d in bad:
        with pytest.raises(SceneError):
            F.parse_scene(d, str(tmp_path))
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(SceneError):
        F.load_scene(str(tmp_path / "bad.json"))
    assert cli.main(["query", "--scene", str(tmp_path / "bad.json"), "--point", "0,0,0"]) == 2
    assert cli.main(["query", "--scene", str(tmp_path / "s.json"), "--point", "0,0"]) == 2


def test_wire_formats_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    w = rng.normal(size=(3, 4, 5)).astype(np.float32)
    F.write_wng1(str(tmp_path / "g.f32"), w)
    raw = (tmp_path / "g.f32").read_bytes()
    assert raw[:4] == b"WNG1" and np.frombuffer(raw[4:16], "<u4").tolist() == [3, 4, 5]
    # x fastest
    assert np.frombuffer(raw[16:20], "<f4")[0] == w[0, 0, 0]
    assert np.frombuffer(raw[20:24], "<f4")[0] == w[1, 0, 0]
    assert np.array_equal(F.read_wng1(str(tmp_path / "g.f32")), w)
    occ = w > 0
    F.write_occupancy(str(tmp_path / "o.bin"), occ)
    assert np.array_equal(F.read_occupancy(str(tmp_path / "o.bin"), occ.shape), occ)
    img = rng.uniform(-0.25, 1.25, (5, 7))
    F.write_pgm16(str(tmp_path / "i.pgm"), img)
    q = F.read_pgm16(str(tmp_path / "i.pgm"))
    assert q.shape == (5, 7)
    assert np.abs(q / 65535.0 * 1.5 - 0.25 - img).max() <= 0.5 * 1.5 / 65535 + 1e-12
    (tmp_path / "q.csv").write_text("x,y,z\n1,2,3\n4, 5, 6\n")
    assert F.read_queries_csv(str(tmp_path / "q.csv")).tolist() == [[1, 2, 3], [4, 5, 6]]
    mx, rmse = F.write_report_csv(str(tmp_path / "r.csv"), [[0, 0, 0], [1, 1, 1]], [1, 0], [1, 0.5])
    assert mx == 0.5 and abs(rmse - np.sqrt(0.125)) < 1e-15


def test_cli_boolean(tmp_path):
    a = np.full((2, 2, 2), 0.5, np.float32)
    F.write_wng1(str(tmp_path / "a.f32"), a)
    F.write_wng1(str(tmp_path / "b.f32"), a)
    F.write_wng1(str(tmp_path / "c.f32"), np.zeros((2, 2, 3), np.float32))
    assert cli.main(["boolean", "--op", "union", str(tmp_path / "a.f32"), str(tmp_path / "b.f32"),
                     "--out", str(tmp_path / "u.f32")]) == 0
    assert np.all(F.read_wng1(str(tmp_path / "u.f32")) == 1.0)
    assert cli.main(["boolean", "--op", "intersection", str(tmp_path / "a.f32"),
                     str(tmp_path / "b.f32"), "--out", str(tmp_path / "i.f32")]) == 0
    assert np.all(F.read_wng1(str(tmp_path / "i.f32")) == 0.25)
    assert cli.main(["boolean", "--op", "union", str(tmp_path / "a.f32"), str(tmp_path / "c.f32"),
                     "--out", str(tmp_path / "x.f32")]) == 2
    (tmp_path / "junk.f32").write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(GridMismatch):
        F.read_wng1(str(tmp_path / "junk.f32"))
