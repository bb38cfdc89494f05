"""ctypes binding of libgwn_b200.so (C ABI: include/gwn_b200.h).

The product path has no CPU fallback: if the in-tree library is missing or
cannot be loaded, every entry point raises :class:`DeviceError` with the
build command.  Build with ``python -m paper_2408_04466_b200.build`` (or
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgwn_b200.so")
# development aid: A/B builds from build.py --variant (build/variants/, git-ignored)
if os.environ.get("GWN_B200_LIB"):
    LIB_PATH = os.environ["GWN_B200_LIB"]

GWN_OK = 0
GWN_E_INVALID = -1
GWN_E_CUDA = -2
GWN_E_NODEVICE = -3
GWN_E_OOM = -4
GWN_HOST_BUFFERS = 1

#: every symbol include/gwn_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "gwn_abi_version", "gwn_last_error", "gwn_params_default", "gwn_scene_create",
    "gwn_scene_destroy", "gwn_scene_info_get", "gwn_eval", "gwn_stats_get", "gwn_set_timing",
    "gwn_all_hits", "gwn_single_loop_batch", "gwn_direction", "gwn_jitter_dir",
    "gwn_net_boundary", "gwn_fp64_peak", "gwn_selftest_rsqrt", "gwn_eval_rays",
    "gwn_solid_angle_many", "gwn_ray_tris_hits", "gwn_release_caches",
)


class GwnParams(C.Structure):
    _fields_ = [
        ("residual", C.c_double), ("dedup", C.c_double), ("tangent", C.c_double),
        ("edge_graze", C.c_double), ("degenerate", C.c_double), ("jitter_scale", C.c_double),
        ("domain_tol", C.c_double), ("t_tol", C.c_double), ("on_surface_t", C.c_double),
        ("band_factor", C.c_double), ("samples_per_edge", C.c_int32), ("max_rounds", C.c_int32),
        ("max_jitters", C.c_int32), ("chunk_queries", C.c_int32), ("dir_seed", C.c_uint64),
        ("cached_rounds", C.c_int32), ("reserved_", C.c_int32),
    ]


class TriBvh(C.Structure):
    """gwn_tri_bvh (include/gwn_b200.h): the reference's Bvh arrays."""
    _fields_ = [("node_min", C.c_void_p), ("node_max", C.c_void_p),
                ("node_left", C.c_void_p), ("node_right", C.c_void_p),
                ("node_start", C.c_void_p), ("node_count", C.c_void_p),
                ("tri_order", C.c_void_p), ("n_nodes", C.c_int64),
                ("V0", C.c_void_p), ("E1", C.c_void_p), ("E2", C.c_void_p),
                ("NN", C.c_void_p), ("NH", C.c_void_p), ("C", C.c_void_p),
                ("R2", C.c_void_p), ("n_tris", C.c_int64)]


class SceneInfo(C.Structure):
    _fields_ = [
        ("n_patches", C.c_int64), ("n_net_edges", C.c_int64), ("n_net_segments", C.c_int64),
        ("bbox_min", C.c_double * 3), ("bbox_max", C.c_double * 3), ("diag", C.c_double),
        ("device", C.c_int32), ("sm_count", C.c_int32), ("n_far_cycles", C.c_int64),
        ("fmm_levels", C.c_int32), ("pad_", C.c_int32), ("fmm_translations", C.c_int64),
        ("fmm_leftover", C.c_int64), ("fmm_build_ms", C.c_double),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("queries", C.c_int64), ("rounds", C.c_int64), ("retried", C.c_int64),
        ("candidates", C.c_int64), ("nodes", C.c_int64), ("newton_iters", C.c_int64),
        ("roots", C.c_int64), ("boundary_segments", C.c_int64), ("kernel_launches", C.c_int64),
        ("ms_cull", C.c_double), ("ms_intersect", C.c_double), ("ms_boundary", C.c_double),
        ("ms_other", C.c_double), ("ms_k3_candidates", C.c_double),
        ("ms_k3_fallback", C.c_double), ("ms_k3_newton", C.c_double),
        ("k3_fallback_items", C.c_int64), ("k3_newton_items", C.c_int64),
        ("far_pairs", C.c_int64), ("far_terms", C.c_int64), ("near_pairs", C.c_int64),
        ("ms_k4_far", C.c_double), ("ms_k4_exact", C.c_double), ("rounds_built", C.c_int64),
        ("ms_round_build", C.c_double), ("local_evals", C.c_int64),
        ("shadow_pairs", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise E.DeviceError(
                f"{LIB_PATH} is not built; run `python -m paper_2408_04466_b200.build` "
                "(nvcc, sm_100a).  There is no CPU fallback.")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - environment specific
            raise E.DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        dp = C.POINTER(C.c_double)
        vp = C.c_void_p
        L.gwn_abi_version.restype = C.c_int
        L.gwn_last_error.restype = C.c_char_p
        L.gwn_params_default.argtypes = [C.POINTER(GwnParams)]
        L.gwn_scene_create.argtypes = [dp, C.c_int64, C.POINTER(GwnParams), C.c_int,
                                       C.POINTER(vp)]
        L.gwn_scene_destroy.argtypes = [vp]
        L.gwn_scene_info_get.argtypes = [vp, C.POINTER(SceneInfo)]
        L.gwn_eval.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, vp, C.c_int32, vp]
        L.gwn_eval_rays.argtypes = [vp, vp, C.c_int64, dp, vp, vp, vp, vp, C.c_int32, vp,
                                    C.POINTER(C.c_int64)]
        L.gwn_stats_get.argtypes = [vp, C.POINTER(Stats)]
        L.gwn_set_timing.argtypes = [vp, C.c_int32]
        L.gwn_all_hits.argtypes = [vp, C.c_int64, dp, dp, C.POINTER(GwnParams), C.c_double,
                                   C.c_double, dp, dp, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int8), C.POINTER(C.c_int8), C.c_int32,
                                   C.POINTER(C.c_int32)]
        L.gwn_single_loop_batch.argtypes = [dp, C.c_int64, dp, dp, dp, C.POINTER(C.c_int64),
                                            C.c_int64, dp, C.c_int64, C.c_double, C.c_double,
                                            dp, C.POINTER(C.c_int8), C.c_int]
        L.gwn_direction.argtypes = [C.c_uint64, C.c_int32, dp]
        L.gwn_jitter_dir.argtypes = [C.c_uint64, C.c_int64, C.c_int32, dp]
        L.gwn_net_boundary.argtypes = [dp, C.c_int64, dp, C.POINTER(C.c_int32)]
        L.gwn_net_boundary.restype = C.c_int64
        L.gwn_fp64_peak.argtypes = [C.c_int, dp, dp]
        L.gwn_selftest_rsqrt.argtypes = [C.c_int, C.c_int64, C.POINTER(C.c_uint64)]
        ip = C.POINTER(C.c_int64)
        L.gwn_solid_angle_many.argtypes = [dp, C.c_int64, ip, C.c_int64, dp, C.c_int64,
                                           C.c_double, dp, C.POINTER(C.c_int8), C.c_int]
        L.gwn_ray_tris_hits.argtypes = [C.POINTER(TriBvh), dp, dp, C.c_int64, C.c_double,
                                        C.c_double, C.c_double, C.c_double, ip, dp, ip, dp,
                                        dp, dp, C.c_int64, C.c_int]
        L.gwn_ray_tris_hits.restype = C.c_int64
        L.gwn_release_caches.argtypes = [C.c_int]
        L.gwn_release_caches.restype = C.c_int
        _lib = L
    return _lib


def check(rc: int, what: str) -> int:
    """Map C-ABI return codes to the GwnError hierarchy (errors.py:9-90)."""
    if rc >= 0:
        return rc
    msg = f"{what}: {lib().gwn_last_error().decode(errors='replace')}"
    if rc == GWN_E_INVALID:
        raise ValueError(msg)
    if rc == GWN_E_OOM:
        raise MemoryError(msg)
    raise E.DeviceError(msg)


def default_params() -> GwnParams:
    p = GwnParams()
    lib().gwn_params_default(C.byref(p))
    return p


def params_from_eps(eps) -> GwnParams:
    """gwn_params with the EpsilonConfig fields the kernels consume
    (config.py:15-38 names -> include/gwn_b200.h fields); engine knobs at
    their defaults."""
    p = default_params()
    p.residual = eps.residual
    p.dedup = eps.dedup
    p.tangent = eps.tangent_parametric
    p.edge_graze = eps.edge_graze
    p.degenerate = eps.degenerate
    p.jitter_scale = eps.jitter_scale
    return p
