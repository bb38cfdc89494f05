"""Top-level engine: the SPEC ``engine`` API on the B200 kernels.

Reference surface (the drop-in boundary):
  * ``Scene`` -- SPEC.md:355-365 (patches + aggregated oriented boundary)
  * ``winding_number(scene, p)`` -- SPEC.md:371-380
  * ``winding_numbers_along_ray(scene, r, ts)`` -- SPEC.md:381-389
  * ``combine(a, b, op)`` -- SPEC.md:409-416
plus the batched call every other path funnels into,
``winding_numbers(scene, queries)``, which is one ``gwn_eval`` of
libgwn_b200.so.  Accepts numpy arrays (host buffers; the library does the
copies) or torch tensors (CUDA tensors stay on the device; CPU tensors,
ideally pinned, are copied inside the call).
"""

from __future__ import annotations

import ctypes as C
import warnings
from typing import Iterable

import numpy as np

from . import _lib
from . import config as cfg
from .config import DEFAULT_EPS, EpsilonConfig
from .errors import (STATUS_ERRORS, STATUS_EXHAUSTED, STATUS_JITTER_EXHAUSTED, STATUS_OK,
                     DegenerateProjection, GridMismatch, SceneError, SeedExhausted)
from .geometry import Aabb, Ray


def _as_ctrl(patches) -> np.ndarray:
    if isinstance(patches, np.ndarray):
        ctrl = patches
    else:
        lst = list(patches)
        if lst and hasattr(lst[0], "control"):
            ctrl = np.stack([np.asarray(p.control, dtype=np.float64) for p in lst]) if lst else \
                np.zeros((0, 4, 4, 3))
        else:
            ctrl = np.asarray(lst, dtype=np.float64).reshape(-1, 4, 4, 3)
    ctrl = np.ascontiguousarray(ctrl, dtype=np.float64)
    if ctrl.ndim != 4 or ctrl.shape[1:] != (4, 4, 3):
        raise SceneError(f"expected (P,4,4,3) bicubic control nets, got {ctrl.shape}")
    if not np.all(np.isfinite(ctrl)):
        raise SceneError("control points must be finite")
    return ctrl


class Scene:
    """Immutable device-resident scene (SPEC.md:216 concurrency model).

    ``patches``: a list of :class:`BicubicPatch` (or anything with a
    ``control`` (4,4,3) array) or a ``(P,4,4,3)`` array.
    """

    def __init__(self, patches, eps: EpsilonConfig = DEFAULT_EPS,
                 samples_per_edge: int = 200, device: int | None = None,
                 max_rounds: int = cfg.MAX_ROUNDS, max_jitters: int = cfg.MAX_JITTERS,
                 dir_seed: int = cfg.DIR_SEED, chunk_queries: int = 0,
                 cached_rounds: int = 4):
        if samples_per_edge < 2:
            raise ValueError("need at least 2 samples per edge")
        self.ctrl = _as_ctrl(patches)
        self.eps = eps
        self.samples_per_edge = samples_per_edge
        if device is None:
            device = _current_device()
        self.device = device
        p = _lib.params_from_eps(eps)
        p.samples_per_edge = samples_per_edge
        p.max_rounds = max_rounds
        p.max_jitters = max_jitters
        p.dir_seed = dir_seed
        p.chunk_queries = chunk_queries
        p.cached_rounds = cached_rounds
        self.params = p
        h = C.c_void_p()
        dp = C.POINTER(C.c_double)
        _lib.check(_lib.lib().gwn_scene_create(self.ctrl.ctypes.data_as(dp), len(self.ctrl),
                                               C.byref(p), device, C.byref(h)),
                   "gwn_scene_create")
        self.handle = h
        info = _lib.SceneInfo()
        _lib.check(_lib.lib().gwn_scene_info_get(h, C.byref(info)), "gwn_scene_info_get")
        self.info = info

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().gwn_scene_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None

    @property
    def n_patches(self) -> int:
        return int(self.info.n_patches)

    @property
    def n_net_segments(self) -> int:
        return int(self.info.n_net_segments)

    @property
    def n_far_cycles(self) -> int:
        """Closed net-boundary cycles with a far-field expansion (DESIGN §2 K4)."""
        return int(self.info.n_far_cycles)

    @property
    def local_expansions(self) -> dict:
        """Round 0's octree of far-field local expansions (DESIGN §2 K4): leaf
        level (0 = none), (box, cycle) translations, entries left to the
        per-query path over all leaves, build time at scene creation."""
        i = self.info
        return {"levels": int(i.fmm_levels), "translations": int(i.fmm_translations),
                "leftover_entries": int(i.fmm_leftover), "build_ms": float(i.fmm_build_ms)}

    @property
    def diag(self) -> float:
        return float(self.info.diag)

    def aabb(self) -> Aabb:
        return Aabb(np.array(self.info.bbox_min[:]), np.array(self.info.bbox_max[:]))

    def stats(self) -> dict:
        s = _lib.Stats()
        _lib.check(_lib.lib().gwn_stats_get(self.handle, C.byref(s)), "gwn_stats_get")
        return s.as_dict()

    def set_timing(self, on: bool) -> None:
        _lib.check(_lib.lib().gwn_set_timing(self.handle, int(bool(on))), "gwn_set_timing")


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _check_out(torch, w, st, n: int, device) -> None:
    """Caller-owned outputs are written through raw pointers: reject anything
    the library could write past or across."""
    if w.dtype != torch.float64 or st.dtype != torch.int8:
        raise ValueError("out=(w, status) must be float64 and int8 tensors")
    if w.numel() < n or st.numel() < n:
        raise ValueError(f"out tensors hold {w.numel()}/{st.numel()} elements, need {n}")
    if not (w.is_contiguous() and st.is_contiguous()):
        raise ValueError("out tensors must be contiguous")
    if w.device != device or st.device != device:
        raise ValueError(f"out tensors must live on {device} like the queries")


def winding_numbers(scene: Scene, queries, *, index_base: int = 0, stream=None,
                    out=None, return_status: bool = True):
    """Generalized winding numbers of many query points (one ``gwn_eval``).

    Returns ``(w, status)``; ``status`` codes: 0 ok, 1 on-surface (jittered),
    2 re-shoot budget exhausted, 3 degenerate projection (jittered), 4 still
    on the surface / boundary after the jitter budget (w unreliable).
    ``out=(w, status)``: caller-owned outputs (float64 / int8, at least n
    elements, contiguous, on the queries' device).
    """
    L = _lib.lib()
    if _is_torch(queries):
        import torch
        q = queries
        if q.dtype != torch.float64 or q.dim() != 2 or q.shape[1] != 3:
            raise ValueError("queries must be an (n,3) float64 tensor")
        q = q.contiguous()
        n = q.shape[0]
        if q.is_cuda and q.device.index != scene.device:
            raise ValueError(f"queries on cuda:{q.device.index}, scene on cuda:{scene.device}")
        if out is not None:
            w, st = out
            _check_out(torch, w, st, n, q.device)
        else:
            w = torch.empty(n, dtype=torch.float64, device=q.device)
            st = torch.empty(n, dtype=torch.int8, device=q.device)
        flags = 0 if q.is_cuda else _lib.GWN_HOST_BUFFERS
        if stream is None and q.is_cuda:
            stream = torch.cuda.current_stream(q.device).cuda_stream
        _lib.check(L.gwn_eval(scene.handle, C.c_void_p(q.data_ptr()), n, index_base,
                              C.c_void_p(w.data_ptr()), C.c_void_p(st.data_ptr()), flags,
                              C.c_void_p(stream or 0)), "gwn_eval")
        return (w, st) if return_status else w
    q = np.ascontiguousarray(queries, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] != 3:
        raise ValueError("queries must have shape (n, 3)")
    n = q.shape[0]
    if out is not None:
        w, st = out
        if not (isinstance(w, np.ndarray) and isinstance(st, np.ndarray)):
            raise ValueError("numpy queries need numpy out=(w, status) arrays")
        if w.dtype != np.float64 or st.dtype != np.int8 or w.ndim != 1 or st.ndim != 1:
            raise ValueError("out=(w, status) must be 1-D float64 and int8 arrays")
        if w.size < n or st.size < n:
            raise ValueError(f"out arrays hold {w.size}/{st.size} elements, need {n}")
        if not (w.flags.c_contiguous and st.flags.c_contiguous and w.flags.writeable
                and st.flags.writeable):
            raise ValueError("out arrays must be writeable and contiguous")
    else:
        w = np.empty(n, np.float64)
        st = np.empty(n, np.int8)
    _lib.check(L.gwn_eval(scene.handle, C.c_void_p(q.ctypes.data), n, index_base,
                          C.c_void_p(w.ctypes.data), C.c_void_p(st.ctypes.data),
                          _lib.GWN_HOST_BUFFERS, C.c_void_p(stream or 0)), "gwn_eval")
    return (w, st) if return_status else w


def winding_number(scene: Scene, p) -> float:
    """w(p).  On-surface / degenerate queries are jittered
    by ``jitter_scale * diag`` (at most 3 times) with a warning; an exhausted
    re-shoot budget raises :class:`SeedExhausted`, a query still on the
    surface after the jitter budget :class:`DegenerateProjection`."""
    w, st = winding_numbers(scene, np.asarray(p, dtype=np.float64).reshape(1, 3))
    code = int(st[0])
    if code == STATUS_EXHAUSTED:
        raise SeedExhausted(f"every ray from {p} was tangent / grazing")
    if code == STATUS_JITTER_EXHAUSTED:
        raise DegenerateProjection(f"{p} stayed on the surface after every jitter")
    if code != STATUS_OK:
        warnings.warn(f"query {p}: {STATUS_ERRORS[code].__name__}; evaluated at a jittered point")
    return float(w[0])


def winding_numbers_rays(scene: Scene, origins, direction, ts, offs, *, stream=None,
                         return_rays: bool = False, check: bool = True):
    """Ray reuse (``gwn_eval_rays``): points ``origins[r] + ts[k] * direction``
    for k in ``[offs[r], offs[r+1])``, one intersection pass per ray r.

    ``ts`` must be ascending within each ray.  Returns ``(w, status)`` over
    the flattened points (plus the number of rays cast if ``return_rays``).
    numpy inputs are host buffers (the library does the copies); CUDA torch
    tensors stay on the device and run on the current torch stream.
    """
    L = _lib.lib()
    d = np.ascontiguousarray(direction, dtype=np.float64).reshape(3)
    cast = C.c_int64(0)
    if _is_torch(ts):
        import torch
        o = origins.to(torch.float64).contiguous().reshape(-1, 3)
        t = ts.to(torch.float64).contiguous().reshape(-1)
        f = offs.to(torch.int64).contiguous().reshape(-1)
        R = o.shape[0]
        if f.shape[0] != R + 1:
            raise ValueError("offs must have R+1 entries")
        dev = t.is_cuda
        if dev != o.is_cuda or dev != f.is_cuda:
            raise ValueError("origins, ts and offs must be on the same device")
        if check:
            fc = f.cpu().numpy() if dev else f.numpy()
            if fc[0] != 0 or fc[-1] != t.shape[0] or np.any(np.diff(fc) < 0):
                raise ValueError("offs must be non-decreasing from 0 to len(ts)")
            seg = torch.repeat_interleave(torch.arange(R, device=t.device), f.diff())
            if bool(((t.diff() < 0) & (seg[1:] == seg[:-1])).any()):
                raise ValueError("ts must be sorted ascending on every ray")
        n = t.shape[0]
        w = torch.empty(n, dtype=torch.float64, device=t.device)
        st = torch.empty(n, dtype=torch.int8, device=t.device)
        if stream is None and dev:
            stream = torch.cuda.current_stream(t.device).cuda_stream
        if R > 0:
            _lib.check(L.gwn_eval_rays(
                scene.handle, C.c_void_p(o.data_ptr()), R, d.ctypes.data_as(C.POINTER(C.c_double)),
                C.c_void_p(t.data_ptr()), C.c_void_p(f.data_ptr()), C.c_void_p(w.data_ptr()),
                C.c_void_p(st.data_ptr()), 0 if dev else _lib.GWN_HOST_BUFFERS,
                C.c_void_p(stream or 0), C.byref(cast)), "gwn_eval_rays")
    else:
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(ts, dtype=np.float64).reshape(-1)
        f = np.ascontiguousarray(offs, dtype=np.int64).reshape(-1)
        R = o.shape[0]
        if f.shape[0] != R + 1 or f[0] != 0 or f[-1] != t.shape[0] or np.any(np.diff(f) < 0):
            raise ValueError("offs must have R+1 non-decreasing entries from 0 to len(ts)")
        if check:
            seg = np.repeat(np.arange(R), np.diff(f))
            if np.any((np.diff(t) < 0) & (seg[1:] == seg[:-1])):
                raise ValueError("ts must be sorted ascending on every ray")
        n = t.shape[0]
        w = np.empty(n, np.float64)
        st = np.empty(n, np.int8)
        if R > 0:
            _lib.check(L.gwn_eval_rays(
                scene.handle, C.c_void_p(o.ctypes.data), R,
                d.ctypes.data_as(C.POINTER(C.c_double)), C.c_void_p(t.ctypes.data),
                C.c_void_p(f.ctypes.data), C.c_void_p(w.ctypes.data), C.c_void_p(st.ctypes.data),
                _lib.GWN_HOST_BUFFERS, C.c_void_p(stream or 0), C.byref(cast)), "gwn_eval_rays")
    scene.rays_cast = int(cast.value)
    return (w, st, int(cast.value)) if return_rays else (w, st)


def _device_torch():
    """torch if a CUDA device is usable (grid generation on the device), else None."""
    try:
        import torch
        return torch if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover
        return None


def winding_numbers_along_ray(scene: Scene, r: Ray, ts: Iterable[float]) -> list[float]:
    """w at r.origin + t r.direction for sorted ts: one
    intersection pass for the ray, chi of every point from the cached hits
    beyond it (``gwn_eval_rays``)."""
    ts = np.asarray(list(ts), dtype=np.float64)
    if ts.size == 0:
        return []
    if np.any(np.diff(ts) < 0):
        raise ValueError("ts must be sorted ascending")
    w, _ = winding_numbers_rays(scene, np.asarray(r.origin, np.float64)[None, :],
                                np.asarray(r.direction, np.float64), ts,
                                np.array([0, ts.size], np.int64))
    return [float(x) for x in w]


def slice(scene: Scene, origin, u_axis, v_axis, width: int, height: int) -> np.ndarray:
    """Winding numbers at the W x H pixel centres of the plane patch
    ``origin + a u_axis + b v_axis``, a, b in [0,1].

    Pixel (j, i) (row j along v, column i along u) is at
    ``origin + (i+0.5)/W u_axis + (j+0.5)/H v_axis``.  The pixels are grouped
    into min(W, H) collinear families along the longer axis, one ray each
    (PAPER.md:305-307); ``scene.rays_cast`` records the count.  Returns an
    (H, W) array.
    """
    W, H = int(width), int(height)
    if W < 1 or H < 1:
        raise ValueError("W, H must be >= 1")
    o = np.asarray(origin, np.float64).reshape(3)
    u = np.asarray(u_axis, np.float64).reshape(3)
    v = np.asarray(v_axis, np.float64).reshape(3)
    along_u = W >= H
    a, b = (u, v) if along_u else (v, u)
    na, nb = (W, H) if along_u else (H, W)
    la = float(np.linalg.norm(a))
    if not la > 0:
        raise ValueError("degenerate slice axes")
    d = a / la
    T = _device_torch()
    if T is not None:
        dev = T.device("cuda", scene.device)
        fb = (T.arange(nb, dtype=T.float64, device=dev) + 0.5) / nb
        origins = T.from_numpy(o).to(dev)[None, :] + fb[:, None] * T.from_numpy(b).to(dev)[None, :]
        ts = ((T.arange(na, dtype=T.float64, device=dev) + 0.5) / na * la).repeat(nb)
        offs = T.arange(nb + 1, dtype=T.int64, device=dev) * na
        w, _ = winding_numbers_rays(scene, origins, d, ts, offs, check=False)
        img = w.reshape(nb, na).cpu().numpy()
    else:
        fb = (np.arange(nb) + 0.5) / nb
        origins = o[None, :] + fb[:, None] * b[None, :]
        ts = np.tile((np.arange(na) + 0.5) / na * la, nb)
        offs = np.arange(nb + 1, dtype=np.int64) * na
        w, _ = winding_numbers_rays(scene, origins, d, ts, offs, check=False)
        img = w.reshape(nb, na)
    return img if along_u else img.T.copy()


def voxelize(scene: Scene, n: int, box_min=None, box_max=None, threshold: float = 0.5):
    """Winding numbers and occupancy at the n^3 voxel centres of
    [box_min, box_max] (default: the scene AABB) with n^2 rays along +x
    (occupied iff w >= threshold, PAPER §7).

    Returns ``(occupancy bool (n,n,n), w (n,n,n))`` indexed [ix, iy, iz];
    ``scene.rays_cast`` == n^2.
    """
    n = int(n)
    if n < 1:
        raise ValueError("N must be >= 1")
    if box_min is None or box_max is None:
        bb = scene.aabb()
        box_min = bb.min_corner if box_min is None else box_min
        box_max = bb.max_corner if box_max is None else box_max
    lo = np.asarray(box_min, np.float64).reshape(3)
    hi = np.asarray(box_max, np.float64).reshape(3)
    T = _device_torch()
    if T is not None:  # grid generated and transposed on the device
        dev = T.device("cuda", scene.device)
        c = (T.arange(n, dtype=T.float64, device=dev) + 0.5) / n
        ys = float(lo[1]) + c * float(hi[1] - lo[1])
        zs = float(lo[2]) + c * float(hi[2] - lo[2])
        Y, Z = T.meshgrid(ys, zs, indexing="ij")  # ray (iy, iz)
        origins = T.stack([T.full_like(Y, float(lo[0])), Y, Z], dim=-1).reshape(-1, 3)
        ts = (c * float(hi[0] - lo[0])).repeat(n * n)
        offs = T.arange(n * n + 1, dtype=T.int64, device=dev) * n
        w, _ = winding_numbers_rays(scene, origins, np.array([1.0, 0.0, 0.0]), ts, offs,
                                    check=False)
        w = w.reshape(n, n, n).permute(2, 0, 1).contiguous().cpu().numpy()
    else:
        c = (np.arange(n) + 0.5) / n
        ys = lo[1] + c * (hi[1] - lo[1])
        zs = lo[2] + c * (hi[2] - lo[2])
        Y, Z = np.meshgrid(ys, zs, indexing="ij")
        origins = np.stack([np.full(n * n, lo[0]), Y.ravel(), Z.ravel()], axis=1)
        ts = np.tile(c * (hi[0] - lo[0]), n * n)
        offs = np.arange(n * n + 1, dtype=np.int64) * n
        w, _ = winding_numbers_rays(scene, origins, np.array([1.0, 0.0, 0.0]), ts, offs,
                                    check=False)
        w = w.reshape(n, n, n).transpose(2, 0, 1).copy()  # (iy, iz, ix) -> (ix, iy, iz)
    return w >= threshold, w


def combine(field_a, field_b, op: str):
    """Boolean combination of winding-number fields."""
    a, b = np.asarray(field_a), np.asarray(field_b)
    if a.shape != b.shape:
        raise GridMismatch(f"grid shapes differ: {a.shape} vs {b.shape}")
    if op == "union":
        return a + b
    if op == "intersection":
        return a * b
    raise ValueError(f"unknown op {op!r}")


def direction(seed: int, rnd: int) -> np.ndarray:
    """Direction of re-shoot round ``rnd`` (host helper, same as the oracle)."""
    d = np.empty(3)
    _lib.lib().gwn_direction(seed, rnd, d.ctypes.data_as(C.POINTER(C.c_double)))
    return d


def net_boundary(ctrl) -> tuple[np.ndarray, np.ndarray]:
    """Net boundary edge curves after exact cancellation: ((E,4,3), weights)."""
    ctrl = _as_ctrl(ctrl)
    L = _lib.lib()
    dp = C.POINTER(C.c_double)
    n = L.gwn_net_boundary(ctrl.ctypes.data_as(dp), len(ctrl), None, None)
    ec = np.empty((max(n, 1), 4, 3))
    w = np.empty(max(n, 1), np.int32)
    L.gwn_net_boundary(ctrl.ctypes.data_as(dp), len(ctrl), ec.ctypes.data_as(dp),
                       w.ctypes.data_as(C.POINTER(C.c_int32)))
    return ec[:n], w[:n]


def release_caches(device: int = 0) -> None:
    """Free this thread's cached eval workspace on `device` (gwn_eval keeps
    its buffers at the largest batch seen for the next call)."""
    _lib.check(_lib.lib().gwn_release_caches(int(device)), "gwn_release_caches")


def fp64_peak(device: int = 0) -> tuple[float, float]:
    """Measured FP64 DFMA peak (TFLOP/s, ms) of ``device``."""
    tf, ms = C.c_double(), C.c_double()
    _lib.check(_lib.lib().gwn_fp64_peak(device, C.byref(tf), C.byref(ms)), "gwn_fp64_peak")
    return tf.value, ms.value
