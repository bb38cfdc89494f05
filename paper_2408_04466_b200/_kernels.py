"""Kernel dispatch layer -- the GPU backend slot of pkg/src/gwn/_kernels.py.

The reference dispatches each hot kernel on ``numba_enabled()``
(_accel.py:28) between a numba and a numpy twin; the batch boundary kernel
``single_loop_batch`` (_kernels.py:801-823) has no numpy twin and returns
``None`` without numba.  This module provides the same call signature backed
by libgwn_b200.so (``gwn_single_loop_batch``): contiguous float64/int64 in,
fresh ``(w, ok)`` out, per-element ``ok`` flags instead of exceptions.

Semantics differ only where the reference gives up: the fan formula handles
self-crossing projections and straight edges, so ``ok == 0`` is returned
only for a hit clash (|t_h - t| <= t_eps, :782-784) or a degenerate
projection (:541-542).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def single_loop_batch(loop_pts, origin, direction, hit_ts, hit_signs, query_ts,
                      on_tol, t_eps, device: int = 0):
    loop = np.ascontiguousarray(loop_pts, dtype=np.float64)
    if loop.ndim != 2 or loop.shape[1] != 3 or len(loop) < 3:
        raise ValueError("loop_pts must be (B>=3, 3)")
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(direction, dtype=np.float64)
    ht = np.ascontiguousarray(hit_ts, dtype=np.float64)
    hs = np.ascontiguousarray(hit_signs, dtype=np.int64)
    qt = np.ascontiguousarray(query_ts, dtype=np.float64)
    K = len(qt)
    w = np.zeros(K, np.float64)
    ok = np.zeros(K, np.int8)
    dp = C.POINTER(C.c_double)
    _lib.check(_lib.lib().gwn_single_loop_batch(
        loop.ctypes.data_as(dp), len(loop), o.ctypes.data_as(dp), d.ctypes.data_as(dp),
        ht.ctypes.data_as(dp), hs.ctypes.data_as(C.POINTER(C.c_int64)), len(ht),
        qt.ctypes.data_as(dp), K, float(on_tol), float(t_eps), w.ctypes.data_as(dp),
        ok.ctypes.data_as(C.POINTER(C.c_int8)), device), "gwn_single_loop_batch")
    return w, ok
