"""Command-line surface over the engine:

    python -m paper_2408_04466_b200 query    --scene S --point x,y,z [--oracle]
    python -m paper_2408_04466_b200 slice    --scene S --origin x,y,z --u x,y,z --v x,y,z
                                             --res WxH --out img.pgm [--range lo,hi]
    python -m paper_2408_04466_b200 voxelize --scene S --res N [--box x0,y0,z0,x1,y1,z1]
                                             [--threshold 0.5] --out grid.f32 [--occ occ.bin]
    python -m paper_2408_04466_b200 boolean  --op union|intersection a.f32 b.f32 --out c.f32
    python -m paper_2408_04466_b200 compare  --scene S --queries q.csv --out report.csv

Exit codes: 0 ok, 2 schema / usage / grid errors, 3 a query still degenerate
(or its re-shoot budget exhausted) after the jitter budget.  Parametric
patches (bicubic, coons, bezier_triangle) run on the ray engine with ray
reuse for slices and voxels; triangle meshes (mesh_obj) add their exact
solid-angle winding numbers (w is additive over surfaces).
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import engine, formats
from .errors import GridMismatch, SceneError, GwnError

EXIT_SCHEMA = 2
EXIT_DEGENERATE = 3


class SceneEval:
    """A loaded SceneFile: the device scene of its parametric patches plus
    its triangle meshes."""

    def __init__(self, spec: formats.SceneSpecFile):
        self.spec = spec
        self.scene = (engine.Scene(spec.ctrl, eps=spec.eps, samples_per_edge=spec.samples_per_edge)
                      if len(spec.ctrl) else None)
        self.meshes = spec.meshes

    def _mesh_w(self, P):
        from .mesh import mesh_winding_numbers
        w = np.zeros(len(P))
        for V, T in self.meshes:
            if len(T):
                w += mesh_winding_numbers(V, T, P)[0]
        return w

    def points(self, P):
        P = np.asarray(P, np.float64).reshape(-1, 3)
        w = np.zeros(len(P))
        st = np.zeros(len(P), np.int8)
        if self.scene is not None and len(P):
            w, st = engine.winding_numbers(self.scene, P)
        return w + self._mesh_w(P), st

    def slice(self, origin, u, v, W, H):
        if self.scene is not None:
            img = engine.slice(self.scene, origin, u, v, W, H)
            rays = self.scene.rays_cast
        else:
            img, rays = np.zeros((H, W)), 0
        if self.meshes:
            jj, ii = np.meshgrid((np.arange(H) + 0.5) / H, (np.arange(W) + 0.5) / W, indexing="ij")
            P = (np.asarray(origin, float) + ii.ravel()[:, None] * np.asarray(u, float)
                 + jj.ravel()[:, None] * np.asarray(v, float))
            img = img + self._mesh_w(P).reshape(H, W)
        return img, rays

    def voxelize(self, n, lo, hi, threshold):
        if self.scene is not None:
            _, w = engine.voxelize(self.scene, n, lo, hi, threshold)
            rays = self.scene.rays_cast
        else:
            w, rays = np.zeros((n, n, n)), 0
        if self.meshes:
            c = (np.arange(n) + 0.5) / n
            ax = [lo[k] + c * (hi[k] - lo[k]) for k in range(3)]
            X, Y, Z = np.meshgrid(*ax, indexing="ij")
            w = w + self._mesh_w(np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)).reshape(n, n, n)
        return w >= threshold, w, rays

    def bbox(self):
        pts = [self.spec.ctrl.reshape(-1, 3)] + [V for V, _ in self.meshes]
        pts = np.concatenate(pts) if pts else np.zeros((1, 3))
        return pts.min(axis=0), pts.max(axis=0)

    def oracle(self, P, tess: int = 64):
        """Direct solid-angle oracle: every parametric patch
        tessellated tess x tess, meshes exactly."""
        from .mesh import mesh_winding_numbers
        w = self._mesh_w(P)
        if len(self.spec.ctrl):
            V, T = tessellate(self.spec.ctrl, tess)
            w = w + mesh_winding_numbers(V, T, P)[0]
        return w


def tessellate(ctrl, n: int):
    """Triangulated n x n grid per bicubic patch (f_u x f_v orientation)."""
    g = np.linspace(0.0, 1.0, n + 1)
    s = 1.0 - g
    B = np.stack([s ** 3, 3 * g * s * s, 3 * g * g * s, g ** 3], axis=1)
    Vs, Ts, base = [], [], 0
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    a0 = (i * (n + 1) + j).ravel()
    b0 = ((i + 1) * (n + 1) + j).ravel()
    for P in np.asarray(ctrl).reshape(-1, 4, 4, 3):
        Vs.append(np.einsum("ui,vj,ijk->uvk", B, B, P).reshape(-1, 3))
        a, b = a0 + base, b0 + base
        Ts.append(np.stack([np.stack([a, b, b + 1], 1), np.stack([a, b + 1, a + 1], 1)], 1)
                  .reshape(-1, 3))
        base += (n + 1) ** 2
    if not Vs:
        return np.zeros((0, 3)), np.zeros((0, 3), np.int64)
    return np.concatenate(Vs), np.concatenate(Ts).astype(np.int64)


def _vec(s: str, n: int = 3):
    try:
        v = [float(x) for x in s.split(",")]
    except ValueError:
        raise SceneError(f"expected {n} comma-separated numbers, got {s!r}") from None
    if len(v) != n:
        raise SceneError(f"expected {n} comma-separated numbers, got {s!r}")
    return np.asarray(v)


def _res(s: str):
    try:
        w, h = (int(x) for x in s.lower().split("x"))
    except ValueError:
        raise SceneError(f"--res must be WxH, got {s!r}") from None
    if w < 1 or h < 1:
        raise SceneError("--res must be at least 1x1")
    return w, h


def cmd_query(a) -> int:
    p = _vec(a.point)
    ev = SceneEval(formats.load_scene(a.scene))
    w, st = ev.points(p[None, :])
    print(f"w={w[0]:.9f}")
    if a.oracle:
        o = ev.oracle(p[None, :], a.tess)[0]
        print(f"oracle={o:.9f} diff={abs(o - w[0]):.3e}")
    return EXIT_DEGENERATE if int(st[0]) in (2, 4) else 0  # budgets spent


def cmd_slice(a) -> int:
    W, H = _res(a.res)
    lo, hi = _vec(a.range, 2) if a.range else (-0.25, 1.25)
    if not hi > lo:
        raise SceneError("--range must have hi > lo")
    o, u, v = _vec(a.origin), _vec(a.u), _vec(a.v)
    ev = SceneEval(formats.load_scene(a.scene))
    img, rays = ev.slice(o, u, v, W, H)
    formats.write_pgm16(a.out, img, lo, hi)
    print(f"rays={rays} min={img.min():.9f} max={img.max():.9f}")
    return 0


def cmd_voxelize(a) -> int:
    if a.res < 1:
        raise SceneError("--res must be >= 1")
    b = _vec(a.box, 6) if a.box else None
    ev = SceneEval(formats.load_scene(a.scene))
    if b is not None:
        lo, hi = b[:3], b[3:]
    else:
        lo, hi = ev.bbox()
    if np.any(hi < lo):
        raise SceneError("--box must have min <= max")
    occ, w, rays = ev.voxelize(a.res, lo, hi, a.threshold)
    formats.write_wng1(a.out, w)
    if a.occ:
        formats.write_occupancy(a.occ, occ)
    print(f"rays={rays} occupied={int(occ.sum())}")
    return 0


def cmd_boolean(a) -> int:
    ga, gb = formats.read_wng1(a.a), formats.read_wng1(a.b)
    formats.write_wng1(a.out, engine.combine(ga, gb, a.op))
    return 0


def cmd_compare(a) -> int:
    P = formats.read_queries_csv(a.queries)
    ev = SceneEval(formats.load_scene(a.scene))
    w, _ = ev.points(P)
    o = ev.oracle(P, a.tess)
    mx, rmse = formats.write_report_csv(a.out, P, o, w)
    print(f"max={mx:.3e} rmse={rmse:.3e} n={len(P)}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2408_04466_b200",
                                 description="B200 generalized winding numbers (SPEC cli)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    q = sub.add_parser("query")
    q.add_argument("--scene", required=True)
    q.add_argument("--point", required=True)
    q.add_argument("--oracle", action="store_true")
    q.add_argument("--tess", type=int, default=64)
    s = sub.add_parser("slice")
    s.add_argument("--scene", required=True)
    s.add_argument("--origin", required=True)
    s.add_argument("--u", required=True)
    s.add_argument("--v", required=True)
    s.add_argument("--res", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("--range")
    v = sub.add_parser("voxelize")
    v.add_argument("--scene", required=True)
    v.add_argument("--res", type=int, required=True)
    v.add_argument("--box")
    v.add_argument("--threshold", type=float, default=0.5)
    v.add_argument("--out", required=True)
    v.add_argument("--occ")
    b = sub.add_parser("boolean")
    b.add_argument("--op", required=True, choices=["union", "intersection"])
    b.add_argument("a")
    b.add_argument("b")
    b.add_argument("--out", required=True)
    c = sub.add_parser("compare")
    c.add_argument("--scene", required=True)
    c.add_argument("--queries", required=True)
    c.add_argument("--out", required=True)
    c.add_argument("--tess", type=int, default=64)
    return ap


_VEC_OPTS = ("--point", "--origin", "--u", "--v", "--box", "--range")


def _join_negative_vectors(argv):
    """`--origin -0.25,0,1`: argparse would read the value as an option;
    glue vector values that start with '-' to their option."""
    out, k = [], 0
    while k < len(argv):
        t = argv[k]
        if t in _VEC_OPTS and k + 1 < len(argv) and argv[k + 1][:1] == "-" and \
                argv[k + 1][1:2] in "0123456789.":
            out.append(f"{t}={argv[k + 1]}")
            k += 2
            continue
        out.append(t)
        k += 1
    return out


def main(argv=None) -> int:
    ap = build_parser()
    argv = _join_negative_vectors(list(sys.argv[1:] if argv is None else argv))
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse usage errors exit 2 already
        return int(e.code) if e.code is not None else EXIT_SCHEMA
    fn = {"query": cmd_query, "slice": cmd_slice, "voxelize": cmd_voxelize,
          "boolean": cmd_boolean, "compare": cmd_compare}[a.cmd]
    try:
        return fn(a)
    except (SceneError, GridMismatch, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_SCHEMA
    except GwnError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DEGENERATE if "SeedExhausted" in type(exc).__name__ else 1


if __name__ == "__main__":
    sys.exit(main())
