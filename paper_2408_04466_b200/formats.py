"""Scene ingestion and wire formats.

* ``SceneFile`` JSON: ``patches[]`` with ``type`` in
  {bicubic, coons, bezier_triangle, mesh_obj, bem_loop}, global
  ``boundary_samples_per_edge`` (default 200) and ``epsilons``.
  Patch types reach the one B200 kernel path by exact conversion:
    - ``bicubic``: a (4,4,3) control net, the north-star type;
    - ``coons`` (surfaces.py:499-553): a bilinearly blended Coons patch of
      four cubic boundary curves IS a bicubic patch; its net is the blend of
      the curves' nets (degree-elevated rulings minus the bilinear corner
      term), so the hull is valid (unlike the reference's curve-only AABB,
      SURVEY P11);
    - ``bezier_triangle`` (surfaces.py:431-476, basis :372-386): the cubic
      triangle composed with (s, t) -> (u, v) = (s (1 - t), t) is a bicubic
      patch with the t = 1 edge collapsed onto the (0,1) corner, same
      orientation (the Jacobian factor is 1 - t >= 0);
    - ``mesh_obj``: a Wavefront OBJ triangle mesh, evaluated exactly by the
      solid-angle kernel (the reference's ground truth);
    - ``bem_loop``: BEM minimal surfaces are out of this tier's scope
       and rejected with a SceneError.
* ``WNG1`` voxel grids: 16-byte header (magic ``WNG1``,
  u32 N x 3), raw little-endian float32, x fastest; occupancy bit-packed,
  x fastest.
* 16-bit PGM slices: linear map of w over [lo, hi].
* Query CSV (one ``x,y,z`` per line, header optional) and the oracle report
  CSV (query xyz, oracle, oneshot, diff).
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from .config import DEFAULT_EPS, EpsilonConfig
from .errors import GridMismatch, SceneError

# ---------------------------------------------------------------------------
# exact conversions to bicubic control nets (ctrl[i, j]: i = u, j = v)
# ---------------------------------------------------------------------------


def coons_to_bicubic(c0, c1, d0, d1, tol: float = 1e-9) -> np.ndarray:
    """(4,4,3) net of the Coons patch of surfaces.py:499-553: ``c0``/``c1``
    along v = 0 / v = 1 (in +u), ``d0``/``d1`` along u = 0 / u = 1 (in +v);
    quadratic curves (3 points) are degree-elevated (surfaces.py:335-343)."""
    cur = []
    for name, c in (("c0", c0), ("c1", c1), ("d0", d0), ("d1", d1)):
        c = np.asarray(c, np.float64)
        if c.shape == (3, 3):
            c = np.array([c[0], (c[0] + 2 * c[1]) / 3, (2 * c[1] + c[2]) / 3, c[2]])
        if c.shape != (4, 3):
            raise SceneError(f"coons curve {name} must have 3 or 4 control points")
        cur.append(c)
    c0, c1, d0, d1 = cur
    p00, p10, p01, p11 = c0[0], c0[3], c1[0], c1[3]
    for a, b in ((c0[0], d0[0]), (c0[3], d1[0]), (c1[0], d0[3]), (c1[3], d1[3])):
        if np.linalg.norm(a - b) > tol:
            raise SceneError("Coons patch corners do not meet within 1e-9")
    net = np.empty((4, 4, 3))
    for i in range(4):
        x = i / 3.0
        for j in range(4):
            y = j / 3.0
            bil = (1 - x) * (1 - y) * p00 + x * (1 - y) * p10 + (1 - x) * y * p01 + x * y * p11
            net[i, j] = (1 - y) * c0[i] + y * c1[i] + (1 - x) * d0[j] + x * d1[j] - bil
    return net


def _tri_to_bicubic_matrix() -> np.ndarray:
    """M (16 x 10) with net[i, j] = sum_k M[4 i + j, k] control[k] for the
    cubic Bezier triangle basis of surfaces.py:372-386 (w = 1 - u - v):
    k: 0 w^3, 1 3vw^2, 2 3uw^2, 3 3v^2w, 4 6uvw, 5 3u^2w, 6 v^3, 7 3uv^2,
    8 3u^2v, 9 u^3.  With u = s (1 - t), v = t, w = (1 - s)(1 - t):
    u^a v^b w^c = [s^a (1-s)^c] [t^b (1-t)^(a+c)], a + b + c = 3, expanded in
    the cubic Bernstein bases of s and t."""
    from math import comb
    terms = [(0, 0, 3, 1), (0, 1, 2, 3), (1, 0, 2, 3), (0, 2, 1, 3), (1, 1, 1, 6),
             (2, 0, 1, 3), (0, 3, 0, 1), (1, 2, 0, 3), (2, 1, 0, 3), (3, 0, 0, 1)]
    M = np.zeros((16, 10))
    for k, (a, b, c, mult) in enumerate(terms):
        # t part: t^b (1-t)^(3-b) = B_b(t) / C(3, b)
        j = b
        ct = 1.0 / comb(3, b)
        # s part: s^a (1-s)^c (s + 1 - s)^(3-a-c) = sum_m C(3-a-c, m) B_{a+m}(s) / C(3, a+m)
        e = 3 - a - c
        for m in range(e + 1):
            i = a + m
            M[4 * i + j, k] += mult * ct * comb(e, m) / comb(3, i)
    return M


_TRI_M = _tri_to_bicubic_matrix()


def bezier_triangle_to_bicubic(control) -> np.ndarray:
    """(4,4,3) net of a cubic Bezier triangle (10 control points,
    surfaces.py:431-476) on the collapsed-edge square parametrisation."""
    C = np.asarray(control, np.float64)
    if C.shape != (10, 3):
        raise SceneError("a cubic Bezier triangle has exactly 10 control points")
    return (_TRI_M @ C).reshape(4, 4, 3)


def bezier_triangle_point(control, u, v):
    """Reference evaluation (surfaces.py:372-386, 449-450), for tests."""
    s = u + v - 1.0
    b = np.array([-s ** 3, 3 * v * s ** 2, 3 * u * s ** 2, -3 * v ** 2 * s, -6 * u * v * s,
                  -3 * u ** 2 * s, v ** 3, 3 * u * v ** 2, 3 * u ** 2 * v, u ** 3])
    return b @ np.asarray(control, np.float64)


# ---------------------------------------------------------------------------
# OBJ meshes
# ---------------------------------------------------------------------------


def read_obj(path: str) -> tuple[np.ndarray, np.ndarray]:
    """Vertices and triangles of a Wavefront OBJ file (``v`` and ``f``
    records; polygons fan-triangulated, ``v/vt/vn`` and negative indices)."""
    V, T = [], []
    try:
        fh = open(path)
    except OSError as exc:
        raise SceneError(f"cannot read OBJ {path}: {exc}") from exc
    with fh:
        for ln, line in enumerate(fh, 1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            try:
                if tok[0] == "v":
                    V.append([float(x) for x in tok[1:4]])
                elif tok[0] == "f":
                    idx = []
                    for t in tok[1:]:
                        k = int(t.split("/")[0])
                        idx.append(k - 1 if k > 0 else len(V) + k)
                    for m in range(1, len(idx) - 1):
                        T.append([idx[0], idx[m], idx[m + 1]])
            except (ValueError, IndexError) as exc:
                raise SceneError(f"{path}:{ln}: malformed OBJ record") from exc
    V = np.asarray(V, np.float64).reshape(-1, 3)
    T = np.asarray(T, np.int64).reshape(-1, 3)
    if T.size and (T.min() < 0 or T.max() >= len(V)):
        raise SceneError(f"{path}: face index out of range")
    return V, T


def write_obj(path: str, V, T) -> None:
    with open(path, "w") as fh:
        for v in np.asarray(V, np.float64):
            fh.write("v %.17g %.17g %.17g\n" % tuple(v))
        for t in np.asarray(T, np.int64):
            fh.write("f %d %d %d\n" % tuple(t + 1))


# ---------------------------------------------------------------------------
# scene files
# ---------------------------------------------------------------------------


@dataclass
class SceneSpecFile:
    """A parsed SceneFile: bicubic nets (all patch types converted) and
    triangle meshes, plus the global options."""
    ctrl: np.ndarray                      # (P,4,4,3)
    meshes: list = field(default_factory=list)   # [(V, T)]
    samples_per_edge: int = 200
    eps: EpsilonConfig = DEFAULT_EPS
    kinds: list = field(default_factory=list)


def _arr(x, shape, what):
    try:
        a = np.asarray(x, np.float64)
    except (TypeError, ValueError) as exc:
        raise SceneError(f"{what}: not numeric") from exc
    if a.shape != shape or not np.all(np.isfinite(a)):
        raise SceneError(f"{what}: expected finite {shape}, got {a.shape}")
    return a


def parse_scene(doc: dict, base_dir: str = ".") -> SceneSpecFile:
    if not isinstance(doc, dict) or not isinstance(doc.get("patches"), list):
        raise SceneError("scene: expected an object with a 'patches' list")
    S = doc.get("boundary_samples_per_edge", 200)
    if not isinstance(S, int) or isinstance(S, bool) or S < 2:
        raise SceneError("boundary_samples_per_edge must be an integer >= 2")
    eps = DEFAULT_EPS
    e = doc.get("epsilons", {})
    if not isinstance(e, dict):
        raise SceneError("epsilons must be an object")
    kw = {}
    for k in ("tangent_parametric", "dedup", "residual", "edge_graze", "degenerate",
              "jitter_scale"):
        if k in e:
            if not isinstance(e[k], (int, float)) or not e[k] > 0:
                raise SceneError(f"epsilons.{k} must be a positive number")
            kw[k] = float(e[k])
    if kw:
        eps = eps.with_(**kw)
    nets, meshes, kinds = [], [], []
    for n, p in enumerate(doc["patches"]):
        if not isinstance(p, dict) or "type" not in p:
            raise SceneError(f"patches[{n}]: missing 'type'")
        t = p["type"]
        if t == "bicubic":
            nets.append(_arr(p.get("control"), (4, 4, 3), f"patches[{n}].control"))
        elif t == "coons":
            if "curves" in p and isinstance(p["curves"], dict):
                cv = p["curves"]
                c = [cv.get(k) for k in ("c0", "c1", "d0", "d1")]
            else:
                c = p.get("control")
                if not isinstance(c, list) or len(c) != 4:
                    raise SceneError(f"patches[{n}]: coons needs 4 curves (c0, c1, d0, d1)")
            if any(x is None for x in c):
                raise SceneError(f"patches[{n}]: coons needs curves c0, c1, d0, d1")
            try:
                nets.append(coons_to_bicubic(*[np.asarray(x, np.float64) for x in c]))
            except (TypeError, ValueError) as exc:
                raise SceneError(f"patches[{n}]: malformed coons curves") from exc
        elif t == "bezier_triangle":
            nets.append(bezier_triangle_to_bicubic(
                _arr(p.get("control"), (10, 3), f"patches[{n}].control")))
        elif t == "mesh_obj":
            path = p.get("path")
            if not isinstance(path, str):
                raise SceneError(f"patches[{n}]: mesh_obj needs a 'path'")
            meshes.append(read_obj(os.path.join(base_dir, path)))
        elif t == "bem_loop":
            raise SceneError(f"patches[{n}]: bem_loop (BEM minimal surfaces) is out of scope")
        else:
            raise SceneError(f"patches[{n}]: unknown type {t!r}")
        kinds.append(t)
    ctrl = np.asarray(nets, np.float64).reshape(-1, 4, 4, 3)
    return SceneSpecFile(ctrl, meshes, S, eps, kinds)


def load_scene(path: str) -> SceneSpecFile:
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except OSError as exc:
        raise SceneError(f"cannot read scene {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise SceneError(f"{path}: malformed JSON: {exc}") from exc
    return parse_scene(doc, os.path.dirname(os.path.abspath(path)))


# ---------------------------------------------------------------------------
# WNG1 voxel grids, occupancy, PGM, CSV
# ---------------------------------------------------------------------------

WNG1_MAGIC = b"WNG1"


def write_wng1(path: str, w) -> None:
    """w indexed [ix, iy, iz] -> header + float32, x fastest."""
    w = np.asarray(w)
    if w.ndim != 3:
        raise ValueError("grid must be 3-D")
    nx, ny, nz = w.shape
    with open(path, "wb") as fh:
        fh.write(WNG1_MAGIC + struct.pack("<3I", nx, ny, nz))
        fh.write(np.ascontiguousarray(w.transpose(2, 1, 0), dtype="<f4").tobytes())


def read_wng1(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        head = fh.read(16)
        if len(head) != 16 or head[:4] != WNG1_MAGIC:
            raise GridMismatch(f"{path}: not a WNG1 grid")
        nx, ny, nz = struct.unpack("<3I", head[4:])
        data = np.frombuffer(fh.read(), dtype="<f4")
    if data.size != nx * ny * nz:
        raise GridMismatch(f"{path}: payload size does not match the header")
    return data.reshape(nz, ny, nx).transpose(2, 1, 0).copy()


def write_occupancy(path: str, occ) -> None:
    occ = np.asarray(occ, bool)
    bits = np.packbits(occ.transpose(2, 1, 0).ravel(), bitorder="little")
    with open(path, "wb") as fh:
        fh.write(bits.tobytes())


def read_occupancy(path: str, shape) -> np.ndarray:
    nx, ny, nz = shape
    bits = np.unpackbits(np.fromfile(path, dtype=np.uint8), bitorder="little")
    return bits[: nx * ny * nz].astype(bool).reshape(nz, ny, nx).transpose(2, 1, 0).copy()


def write_pgm16(path: str, img, lo: float = -0.25, hi: float = 1.25) -> None:
    """16-bit binary PGM, row 0 at the top, linear map of [lo, hi]."""
    img = np.asarray(img, np.float64)
    if not hi > lo:
        raise ValueError("range must have hi > lo")
    q = np.clip(np.rint((img - lo) / (hi - lo) * 65535.0), 0, 65535).astype(">u2")
    h, wd = q.shape
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n65535\n" % (wd, h))
        fh.write(q.tobytes())


def read_pgm16(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        data = fh.read()
    parts = data.split(maxsplit=4)
    if parts[0] != b"P5":
        raise ValueError("not a binary PGM")
    wd, h, mx = int(parts[1]), int(parts[2]), int(parts[3])
    if mx != 65535:
        raise ValueError("not a 16-bit PGM")
    return np.frombuffer(parts[4][: 2 * wd * h], dtype=">u2").reshape(h, wd).astype(np.uint16)


def read_queries_csv(path: str) -> np.ndarray:
    rows = []
    try:
        fh = open(path)
    except OSError as exc:
        raise SceneError(f"cannot read queries {path}: {exc}") from exc
    with fh:
        for ln, line in enumerate(fh, 1):
            s = line.strip()
            if not s:
                continue
            parts = [x.strip() for x in s.split(",")]
            try:
                rows.append([float(x) for x in parts[:3]])
            except ValueError:
                if ln == 1:
                    continue  # header
                raise SceneError(f"{path}:{ln}: expected x,y,z") from None
    return np.asarray(rows, np.float64).reshape(-1, 3)


def write_report_csv(path: str, P, oracle, oneshot) -> tuple[float, float]:
    P = np.asarray(P, np.float64)
    d = np.abs(np.asarray(oneshot) - np.asarray(oracle))
    with open(path, "w") as fh:
        fh.write("x,y,z,oracle,oneshot,diff\n")
        for p, a, b, e in zip(P, oracle, oneshot, d):
            fh.write("%.17g,%.17g,%.17g,%.17g,%.17g,%.3e\n" % (p[0], p[1], p[2], a, b, e))
    mx = float(d.max()) if d.size else 0.0
    rmse = float(np.sqrt(np.mean(d * d))) if d.size else 0.0
    return mx, rmse
