"""Ray and Aabb: the two geometry types of the reference's patch protocol
(pkg/src/gwn/geometry.py: Ray :44-54, Aabb :57-84).  They are interface
types only -- the batched path never builds Python rays, and the slab clip
(geometry.py:198-219) is the K2 cull on the device (csrc/gwn_cull.cu)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import DEFAULT_EPS

Vec3 = np.ndarray


@dataclass(frozen=True)
class Ray:
    """origin + t * direction; the direction is stored unit length
    (the reference re-normalises when | |d| - 1 | > eps.unit_norm)."""

    origin: Vec3
    direction: Vec3

    def __post_init__(self):
        o = np.asarray(self.origin, dtype=np.float64).reshape(3)
        d = np.asarray(self.direction, dtype=np.float64).reshape(3)
        n = float(np.linalg.norm(d))
        if n == 0.0:
            raise ZeroDivisionError("ray direction is the zero vector")
        if abs(n - 1.0) > DEFAULT_EPS.unit_norm:
            d = d / n
        object.__setattr__(self, "origin", o)
        object.__setattr__(self, "direction", d)

    def at(self, t: float) -> Vec3:
        return self.origin + t * self.direction


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box; ValueError when a min coordinate exceeds its max."""

    min_corner: Vec3
    max_corner: Vec3

    def __post_init__(self):
        lo = np.asarray(self.min_corner, dtype=np.float64).reshape(3)
        hi = np.asarray(self.max_corner, dtype=np.float64).reshape(3)
        if (lo > hi).any():
            raise ValueError("Aabb min corner must be <= max corner componentwise")
        object.__setattr__(self, "min_corner", lo)
        object.__setattr__(self, "max_corner", hi)

    @property
    def diag(self) -> float:
        return float(np.linalg.norm(self.max_corner - self.min_corner))

    @staticmethod
    def of_points(points: np.ndarray) -> "Aabb":
        p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        return Aabb(p.min(axis=0), p.max(axis=0))
