"""B200-native batched generalized winding numbers for bicubic Bezier patches.

Drop-in for the reference's (arXiv 2408.04466) query path: patches in, query
points in, winding numbers out -- the SPEC engine API over the reference
patch protocol, running on hand-written sm_100a kernels in libgwn_b200.so.
"""

from .config import DEFAULT_EPS, EpsilonConfig
from .engine import (Scene, combine, direction, fp64_peak, net_boundary, release_caches,
                     winding_number,
                     winding_numbers, winding_numbers_along_ray, winding_numbers_rays,
                     slice, voxelize)
from .errors import GwnError
from .geometry import Aabb, Ray
from .surfaces import BicubicPatch, BoundaryLoop, IntersectionRecord, patch_boundary
from .mesh import build_bvh, intersect_ray_mesh, mesh_winding_numbers

__all__ = [
    "DEFAULT_EPS", "EpsilonConfig", "Scene", "combine", "direction", "fp64_peak", "release_caches",
    "net_boundary", "winding_number", "winding_numbers", "winding_numbers_along_ray",
    "winding_numbers_rays", "slice", "voxelize",
    "GwnError", "Aabb", "Ray", "BicubicPatch", "BoundaryLoop", "IntersectionRecord",
    "patch_boundary", "build_bvh", "intersect_ray_mesh", "mesh_winding_numbers",
]
