"""GPU: the SPEC command line end to end (SPEC.md:591-650 examples) and the
converted patch types (coons, bezier_triangle) against the direct
solid-angle oracle."""

import json
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_04466_b200 import cli, formats as F, scenes  # noqa: E402


def cube_scene(tmp_path, extra=()):
    doc = {"patches": [{"type": "bicubic", "control": c.tolist()} for c in scenes.unit_cube()]
           + list(extra)}
    path = tmp_path / "cube.json"
    path.write_text(json.dumps(doc))
    return str(path)


def run(capsys, *args):
    rc = cli.main(list(args))
    return rc, capsys.readouterr().out


def test_query_and_oracle(tmp_path, capsys):
    s = cube_scene(tmp_path)
    rc, out = run(capsys, "query", "--scene", s, "--point", "0.3,0.6,0.45")
    assert rc == 0 and out.strip() == "w=1.000000000"
    rc, out = run(capsys, "query", "--scene", s, "--point", "3,0.6,0.45", "--oracle")
    assert rc == 0 and out.splitlines()[0] == "w=0.000000000"
    assert float(out.split("diff=")[1]) < 1e-12


def test_slice_rays_and_image(tmp_path, capsys):
    s = cube_scene(tmp_path)
    rc, out = run(capsys, "slice", "--scene", s, "--origin", "-0.25,-0.25,0.5", "--u", "1.5,0,0",
                  "--v", "0,1.5,0", "--res", "3x5", "--out", str(tmp_path / "a.pgm"))
    assert rc == 0 and out.startswith("rays=3 ")
    rc, out = run(capsys, "slice", "--scene", s, "--origin", "-0.25,-0.25,0.5", "--u", "1.5,0,0",
                  "--v", "0,1.5,0", "--res", "32x32", "--out", str(tmp_path / "b.pgm"),
                  "--range", "0,1")
    img = F.read_pgm16(str(tmp_path / "b.pgm"))
    c = -0.25 + (np.arange(32) + 0.5) / 32 * 1.5
    inside = ((c[:, None] > 0) & (c[:, None] < 1)) & ((c[None, :] > 0) & (c[None, :] < 1))
    assert np.array_equal(img, np.where(inside, 65535, 0))
    # fully outside the scene: uniform w = 0
    rc, out = run(capsys, "slice", "--scene", s, "--origin", "5,5,5", "--u", "1,0,0",
                  "--v", "0,1,0", "--res", "4x4", "--out", str(tmp_path / "c.pgm"))
    assert len(np.unique(F.read_pgm16(str(tmp_path / "c.pgm")))) == 1


def test_voxelize_and_boolean(tmp_path, capsys):
    s = cube_scene(tmp_path)
    rc, out = run(capsys, "voxelize", "--scene", s, "--res", "2", "--box", "0,0,0,1,1,1",
                  "--out", str(tmp_path / "g.f32"), "--occ", str(tmp_path / "o.bin"))
    assert rc == 0 and out.strip() == "rays=4 occupied=8"
    assert (tmp_path / "g.f32").read_bytes()[:4] == b"WNG1"
    assert F.read_occupancy(str(tmp_path / "o.bin"), (2, 2, 2)).all()
    rc, out = run(capsys, "voxelize", "--scene", s, "--res", "2", "--box", "0,0,0,1,1,1",
                  "--threshold", "1.5", "--out", str(tmp_path / "h.f32"))
    assert out.strip() == "rays=4 occupied=0"
    rc, _ = run(capsys, "boolean", "--op", "union", str(tmp_path / "g.f32"),
                str(tmp_path / "g.f32"), "--out", str(tmp_path / "u.f32"))
    assert rc == 0 and np.all(F.read_wng1(str(tmp_path / "u.f32")) == 2.0)
    # module entry point, separate process
    r = subprocess.run([sys.executable, "-m", "paper_2408_04466_b200", "query", "--scene", s,
                        "--point", "0.5,0.5,0.5"], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "w=1.000000000"


def test_compare_and_mixed_scene(tmp_path, capsys):
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]) + 3.0
    T = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]])
    F.write_obj(str(tmp_path / "tet.obj"), V, T)
    s = cube_scene(tmp_path, [{"type": "mesh_obj", "path": "tet.obj"}])
    q = tmp_path / "q.csv"
    rng = np.random.default_rng(2)
    P = np.concatenate([rng.uniform(0.05, 0.95, (10, 3)), 3.0 + np.full((1, 3), 0.1),
                        rng.uniform(6, 7, (5, 3))])
    q.write_text("x,y,z\n" + "\n".join(",".join("%.17g" % x for x in p) for p in P))
    rc, out = run(capsys, "compare", "--scene", s, "--queries", str(q), "--out",
                  str(tmp_path / "r.csv"))
    assert rc == 0 and float(out.split("max=")[1].split()[0]) < 1e-9
    rows = np.loadtxt(str(tmp_path / "r.csv"), delimiter=",", skiprows=1)
    assert np.allclose(rows[:, 4], [1.0] * 10 + [1.0] + [0.0] * 5, atol=1e-9)  # cube + tet
    rc, _ = run(capsys, "compare", "--scene", s, "--queries", str(tmp_path / "none.csv"),
                "--out", str(tmp_path / "x.csv"))
    assert rc == 2


def test_coons_and_triangle_patches_vs_tessellation(tmp_path, capsys):
    rng = np.random.default_rng(5)
    c0, c1, d0, d1 = (rng.normal(scale=0.3, size=(4, 3)) + np.array([0, 0, 0.0]) for _ in range(4))
    for k in range(4):
        c0[k] += [k / 3, 0, 0]; c1[k] += [k / 3, 1, 0]; d0[k] += [0, k / 3, 0]; d1[k] += [1, k / 3, 0]
    d0[0], d1[0], d0[3], d1[3] = c0[0], c0[3], c1[0], c1[3]
    tri = np.array([[0, 0, 0], [0, 1 / 3, 0.2], [1 / 3, 0, -0.1], [0, 2 / 3, 0.1], [1 / 3, 1 / 3, 0.3],
                    [2 / 3, 0, 0.0], [0, 1, 0], [1 / 3, 2 / 3, 0.1], [2 / 3, 1 / 3, -0.2], [1, 0, 0]])
    doc = {"boundary_samples_per_edge": 2000, "patches": [
        {"type": "coons", "curves": {"c0": c0.tolist(), "c1": c1.tolist(), "d0": d0.tolist(),
                                     "d1": d1.tolist()}},
        {"type": "bezier_triangle", "control": (tri + [0, 0, 2.0]).tolist()}]}
    (tmp_path / "p.json").write_text(json.dumps(doc))
    q = tmp_path / "q.csv"
    P = np.concatenate([rng.uniform(-0.3, 1.3, (40, 3)) * [1, 1, 0.5] + [0, 0, 0.2],
                        rng.uniform(0, 0.6, (20, 3)) * [1, 1, 0] + [0, 0, 2.35]])
    q.write_text("\n".join(",".join("%.17g" % x for x in p) for p in P))
    rc, out = run(capsys, "compare", "--scene", str(tmp_path / "p.json"), "--queries", str(q),
                  "--out", str(tmp_path / "r.csv"), "--tess", "256")
    # SPEC.md:634 "Bezier patch at 2000 boundary samples vs tessellation oracle < 1e-4"
    assert rc == 0 and float(out.split("max=")[1].split()[0]) < 1e-4
