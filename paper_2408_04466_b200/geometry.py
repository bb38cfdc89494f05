"""Rays and boxes -- the subset of pkg/src/gwn/geometry.py the patch protocol
uses (Ray :44-54, Aabb :57-84, ray_aabb_clip :198-219).  Host-side helpers;
the batched path never builds Python rays."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import DEFAULT_EPS

Vec3 = np.ndarray


def vec(x: float, y: float, z: float) -> Vec3:
    return np.array([x, y, z], dtype=np.float64)


def norm(v: Vec3) -> float:
    return float(np.sqrt(v @ v))


def normalize(v: Vec3) -> Vec3:
    n = norm(v)
    if n == 0.0:
        raise ZeroDivisionError("cannot normalize the zero vector")
    return v / n


def is_unit(v: Vec3, tol: float = DEFAULT_EPS.unit_norm) -> bool:
    return abs(norm(v) - 1.0) <= tol


@dataclass(frozen=True)
class Ray:
    origin: Vec3
    direction: Vec3  # unit (geometry.py:49-51 normalises otherwise)

    def __post_init__(self):
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=np.float64))
        d = np.asarray(self.direction, dtype=np.float64)
        if not is_unit(d):
            d = normalize(d)
        object.__setattr__(self, "direction", d)

    def at(self, t: float) -> Vec3:
        return self.origin + t * self.direction


@dataclass(frozen=True)
class Aabb:
    min_corner: Vec3
    max_corner: Vec3

    def __post_init__(self):
        if np.any(self.min_corner > self.max_corner):
            raise ValueError("Aabb min corner must be <= max corner componentwise")

    @property
    def diag(self) -> float:
        return norm(self.max_corner - self.min_corner)

    @staticmethod
    def of_points(points: np.ndarray) -> "Aabb":
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        return Aabb(pts.min(axis=0), pts.max(axis=0))

    def union(self, other: "Aabb") -> "Aabb":
        return Aabb(np.minimum(self.min_corner, other.min_corner),
                    np.maximum(self.max_corner, other.max_corner))

    def contains(self, p: Vec3, slack: float = 0.0) -> bool:
        return bool(np.all(p >= self.min_corner - slack) and np.all(p <= self.max_corner + slack))


def ray_aabb_clip(r: Ray, box: Aabb) -> tuple[float, float] | None:
    """Slab-method window of the ray inside the box, cut to t >= 0."""
    t_min, t_max = 0.0, np.inf
    for k in range(3):
        o, d = r.origin[k], r.direction[k]
        lo, hi = box.min_corner[k], box.max_corner[k]
        if d == 0.0:
            if o < lo or o > hi:
                return None
            continue
        inv = 1.0 / d
        t0, t1 = (lo - o) * inv, (hi - o) * inv
        if t0 > t1:
            t0, t1 = t1, t0
        t_min = max(t_min, t0)
        t_max = min(t_max, t1)
        if t_max < t_min:
            return None
    return (t_min, t_max)
