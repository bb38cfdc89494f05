"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs, as the checker or the timed CPU
baseline.  The product package ``paper_2408_04466_b200`` never imports this.
See gwn_oracle.h for what is restated from which reference file:line.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgwn_oracle.so")


class Params(C.Structure):
    _fields_ = [
        ("residual", C.c_double), ("dedup", C.c_double), ("tangent", C.c_double),
        ("edge_graze", C.c_double), ("degenerate", C.c_double),
        ("jitter_scale", C.c_double), ("domain_tol", C.c_double), ("t_tol", C.c_double),
        ("on_surface_t", C.c_double), ("band_factor", C.c_double),
        ("samples_per_edge", C.c_int32), ("max_rounds", C.c_int32),
        ("max_jitters", C.c_int32), ("subdiv_depth", C.c_int32), ("dir_seed", C.c_uint64),
    ]


class Record(C.Structure):
    _fields_ = [("t", C.c_double), ("u", C.c_double), ("v", C.c_double),
                ("normal", C.c_double * 3), ("sign", C.c_int32), ("tangency", C.c_int32),
                ("grazing", C.c_int32), ("pad", C.c_int32)]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gwn_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        L.or_params_default.argtypes = [C.POINTER(Params)]
        L.or_ray_aabb_clip.argtypes = [dp, dp, dp, dp, dp, dp]
        L.or_ray_aabb_clip.restype = C.c_int
        L.or_multistart_hits.argtypes = [dp, dp, dp, C.POINTER(Params), C.POINTER(Record), C.c_int]
        L.or_patch_all_hits.argtypes = [dp, dp, dp, C.POINTER(Params), C.POINTER(Record), C.c_int]
        L.or_patch_boundary.argtypes = [dp, C.c_int, dp]
        L.or_loop_fan.argtypes = [dp, C.c_int64, dp, dp]
        L.or_loop_fan.restype = C.c_double
        L.or_net_boundary.argtypes = [dp, C.c_int64, dp, C.POINTER(C.c_int32)]
        L.or_net_boundary.restype = C.c_int64
        L.or_sample_edge.argtypes = [dp, C.c_int, dp]
        L.or_direction.argtypes = [C.c_uint64, C.c_int32, dp]
        L.or_jitter_dir.argtypes = [C.c_uint64, C.c_int64, C.c_int32, dp]
        L.or_scene_eval.argtypes = [dp, C.c_int64, dp, C.POINTER(C.c_int64), C.c_int64,
                                    C.POINTER(Params), dp, C.POINTER(C.c_int8),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int]
        L.or_scene_eval_dir.argtypes = [dp, C.c_int64, dp, C.c_int64, dp, C.POINTER(Params),
                                        C.POINTER(C.c_int32), dp, C.POINTER(C.c_int32), C.c_int]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def params(**kw) -> Params:
    p = Params()
    lib().or_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def ray_aabb_clip(o, d, lo, hi):
    o, d, lo, hi = map(_f64, (o, d, lo, hi))
    t0, t1 = C.c_double(), C.c_double()
    ok = lib().or_ray_aabb_clip(_dp(o), _dp(d), _dp(lo), _dp(hi), C.byref(t0), C.byref(t1))
    return (t0.value, t1.value) if ok else None


@dataclass
class Hit:
    t: float
    u: float
    v: float
    normal: tuple
    sign: int
    tangency: bool
    grazing: bool


def _hits(fn, ctrl, o, d, prm):
    ctrl, o, d = _f64(ctrl), _f64(o), _f64(d)
    buf = (Record * 64)()
    n = fn(_dp(ctrl), _dp(o), _dp(d), C.byref(prm or params()), buf, 64)
    return [Hit(r.t, r.u, r.v, tuple(r.normal), r.sign, bool(r.tangency), bool(r.grazing))
            for r in buf[:n]]


def multistart_hits(ctrl, o, d, prm=None):
    return _hits(lib().or_multistart_hits, ctrl, o, d, prm)


def patch_all_hits(ctrl, o, d, prm=None):
    return _hits(lib().or_patch_all_hits, ctrl, o, d, prm)


def patch_boundary(ctrl, S=200) -> np.ndarray:
    ctrl = _f64(ctrl)
    out = np.empty((4 * (S - 1), 3))
    lib().or_patch_boundary(_dp(ctrl), S, _dp(out))
    return out


def loop_fan(loop, p, d) -> float:
    loop, p, d = _f64(loop), _f64(p), _f64(d)
    return lib().or_loop_fan(_dp(loop), len(loop), _dp(p), _dp(d))


def net_boundary(ctrl):
    ctrl = _f64(ctrl)
    n = lib().or_net_boundary(_dp(ctrl), len(ctrl), None, None)
    ec = np.empty((max(n, 1), 4, 3))
    w = np.empty(max(n, 1), np.int32)
    lib().or_net_boundary(_dp(ctrl), len(ctrl), _dp(ec), w.ctypes.data_as(C.POINTER(C.c_int32)))
    return ec[:n], w[:n]


def sample_edge(ctrl4, S=200) -> np.ndarray:
    ctrl4 = _f64(ctrl4)
    out = np.empty((S, 3))
    lib().or_sample_edge(_dp(ctrl4), S, _dp(out))
    return out


def direction(seed: int, rnd: int) -> np.ndarray:
    d = np.empty(3)
    lib().or_direction(seed, rnd, _dp(d))
    return d


def jitter_dir(seed: int, qidx: int, attempt: int) -> np.ndarray:
    v = np.empty(3)
    lib().or_jitter_dir(seed, qidx, attempt, _dp(v))
    return v


def scene_eval(ctrl, queries, prm=None, qidx=None, nthreads=0):
    ctrl, queries = _f64(ctrl), _f64(queries)
    n = len(queries)
    w = np.empty(n)
    st = np.empty(n, np.int8)
    chi = np.empty(n, np.int32)
    rounds = np.empty(n, np.int32)
    qp = None
    if qidx is not None:
        qidx = np.ascontiguousarray(qidx, dtype=np.int64)
        qp = qidx.ctypes.data_as(C.POINTER(C.c_int64))
    lib().or_scene_eval(_dp(ctrl), len(ctrl), _dp(queries), qp, n, C.byref(prm or params()),
                        _dp(w), st.ctypes.data_as(C.POINTER(C.c_int8)),
                        chi.ctypes.data_as(C.POINTER(C.c_int32)),
                        rounds.ctypes.data_as(C.POINTER(C.c_int32)), nthreads)
    return w, st, chi, rounds


def scene_eval_dir(ctrl, queries, d, prm=None, nthreads=0):
    ctrl, queries, d = _f64(ctrl), _f64(queries), _f64(d)
    n = len(queries)
    chi = np.empty(n, np.int32)
    bt = np.empty(n)
    fl = np.empty(n, np.int32)
    lib().or_scene_eval_dir(_dp(ctrl), len(ctrl), _dp(queries), n, _dp(d),
                            C.byref(prm or params()), chi.ctypes.data_as(C.POINTER(C.c_int32)),
                            _dp(bt), fl.ctypes.data_as(C.POINTER(C.c_int32)), nthreads)
    return chi, bt, fl
