// gwn_patch.cuh -- device helpers for projected bicubic nets (K3).
//
// A node net is the (a, b) pair of 4x4 ray-frame coordinates of a sub-patch
// minus the query's projection, index 4*i+j with i the u index.
#pragma once

#include <stddef.h>

#include "gwn_internal.h"

namespace gwn {

constexpr int kMaxLevel = 44;
constexpr int kNodeBudget = 4096;
constexpr int kNewtonMax = 16;

__device__ __forceinline__ void bern3(double t, double b[4], double db[4]) {
  double s = 1.0 - t;
  b[0] = s * s * s;
  b[1] = 3.0 * t * s * s;
  b[2] = 3.0 * t * t * s;
  b[3] = t * t * t;
  db[0] = -3.0 * s * s;
  db[1] = 3.0 * s * (s - 2.0 * t);
  db[2] = 3.0 * t * (2.0 * s - t);
  db[3] = 3.0 * t * t;
}

// value and partials of one projected coordinate net X (16) at (u,v)
__device__ __forceinline__ void eval_coord(const double* __restrict__ X, const double bu[4],
                                           const double dbu[4], const double bv[4],
                                           const double dbv[4], double& f, double& fu,
                                           double& fv) {
  double r[4], rv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r[i] = bv[0] * X[4 * i] + bv[1] * X[4 * i + 1] + bv[2] * X[4 * i + 2] + bv[3] * X[4 * i + 3];
    rv[i] = dbv[0] * X[4 * i] + dbv[1] * X[4 * i + 1] + dbv[2] * X[4 * i + 2] +
            dbv[3] * X[4 * i + 3];
  }
  f = bu[0] * r[0] + bu[1] * r[1] + bu[2] * r[2] + bu[3] * r[3];
  fu = dbu[0] * r[0] + dbu[1] * r[1] + dbu[2] * r[2] + dbu[3] * r[3];
  fv = bu[0] * rv[0] + bu[1] * rv[1] + bu[2] * rv[2] + bu[3] * rv[3];
}

// de Casteljau halving of 4 values: (p0..p3) -> left in p, right in q
__device__ __forceinline__ void half4(double& p0, double& p1, double& p2, double& p3, double& q0,
                                      double& q1, double& q2, double& q3) {
  double a01 = 0.5 * (p0 + p1), a12 = 0.5 * (p1 + p2), a23 = 0.5 * (p2 + p3);
  double b0 = 0.5 * (a01 + a12), b1 = 0.5 * (a12 + a23);
  double c = 0.5 * (b0 + b1);
  q3 = p3; q2 = a23; q1 = b1; q0 = c;
  p1 = a01; p2 = b0; p3 = c;
}

// Split net (a,b) along u (dir 0) or v (dir 1); left half stays in (a,b),
// right half is written to (ra, rb).
__device__ __forceinline__ void split_net(double* a, double* b, double* ra, double* rb, int dir) {
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    int i0 = dir == 0 ? l : 4 * l;
    int st = dir == 0 ? 4 : 1;
    half4(a[i0], a[i0 + st], a[i0 + 2 * st], a[i0 + 3 * st], ra[i0], ra[i0 + st],
          ra[i0 + 2 * st], ra[i0 + 3 * st]);
    half4(b[i0], b[i0 + st], b[i0 + 2 * st], b[i0 + 3 * st], rb[i0], rb[i0 + st],
          rb[i0 + 2 * st], rb[i0 + 3 * st]);
  }
}

__device__ __forceinline__ bool box_has_origin(const double* a, const double* b, double eps) {
  double amin = a[0], amax = a[0], bmin = b[0], bmax = b[0];
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    amin = fmin(amin, a[k]); amax = fmax(amax, a[k]);
    bmin = fmin(bmin, b[k]); bmax = fmax(bmax, b[k]);
  }
  return amin <= eps && amax >= -eps && bmin <= eps && bmax >= -eps;
}

// Query-independent part of the Krawczyk operator of a node net (local
// coords t in [0,1]^2, centre 1/2):
//   G  = value at the centre, Ys = J(c)^-1 (Newton step = Ys g),
//   R  = radius of (I - J(c)^-1 J(D))(D - c) from the Bernstein hulls of the
//        derivative nets.
// For parallel rays only g(c) = G - q depends on the query, so G, Ys, R of a
// sub-patch can be computed once per direction.
struct KrawPre {
  double Ga, Gb;
  double Y00, Y01, Y10, Y11;
  double R0, R1;
  bool ok;
};

__device__ __forceinline__ KrawPre kraw_pre(const double* a, const double* b) {
  const double w3[4] = {0.125, 0.375, 0.375, 0.125};
  const double w2[3] = {0.25, 0.5, 0.25};
  KrawPre k;
  double ga = 0.0, gb = 0.0, Jua = 0.0, Jub = 0.0, Jva = 0.0, Jvb = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double w = w3[i] * w3[j];
      ga += w * a[4 * i + j];
      gb += w * b[4 * i + j];
      if (i < 3) {
        double wu = w2[i] * w3[j];
        Jua += wu * (a[4 * (i + 1) + j] - a[4 * i + j]);
        Jub += wu * (b[4 * (i + 1) + j] - b[4 * i + j]);
      }
      if (j < 3) {
        double wv = w3[i] * w2[j];
        Jva += wv * (a[4 * i + j + 1] - a[4 * i + j]);
        Jvb += wv * (b[4 * i + j + 1] - b[4 * i + j]);
      }
    }
  }
  k.Ga = ga;
  k.Gb = gb;
  // derivative nets are 3 x differences: J(c) = 3 Jd, Y = Jd^-1 bounds the
  // preconditioned derivative hull, Ys = Y / 3 is the Newton step matrix
  const double det = Jua * Jvb - Jva * Jub;
  k.ok = fabs(det) > 1e-300 && isfinite(det);
  if (!k.ok) {
    k.Y00 = k.Y01 = k.Y10 = k.Y11 = 0.0;
    k.R0 = k.R1 = INFINITY;
    return k;
  }
  const double id = 1.0 / det;
  const double Y00 = Jvb * id, Y01 = -Jva * id, Y10 = -Jub * id, Y11 = Jua * id;
  double e11 = 0.0, e21 = 0.0, e12 = 0.0, e22 = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double qa = a[4 * (i + 1) + j] - a[4 * i + j], qb = b[4 * (i + 1) + j] - b[4 * i + j];
      e11 = fmax(e11, fabs(Y00 * qa + Y01 * qb - 1.0));
      e21 = fmax(e21, fabs(Y10 * qa + Y11 * qb));
    }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double qa = a[4 * i + j + 1] - a[4 * i + j], qb = b[4 * i + j + 1] - b[4 * i + j];
      e12 = fmax(e12, fabs(Y00 * qa + Y01 * qb));
      e22 = fmax(e22, fabs(Y10 * qa + Y11 * qb - 1.0));
    }
  // rounding + 1e-7 box expansion margins
  const double rad = 0.5 + 1e-7;
  k.R0 = (e11 + e12) * rad * (1.0 + 1e-9) + 1e-12;
  k.R1 = (e21 + e22) * rad * (1.0 + 1e-9) + 1e-12;
  k.Y00 = Y00 * (1.0 / 3.0);
  k.Y01 = Y01 * (1.0 / 3.0);
  k.Y10 = Y10 * (1.0 / 3.0);
  k.Y11 = Y11 * (1.0 / 3.0);
  return k;
}

// Separating-axis test of the point q against the convex hull of a node net
// along the normals of its two centre tangent directions (u and v partials,
// difference form).  Returns false if q is provably outside the hull.
__device__ __forceinline__ bool hull_sat(const double* a, const double* b, double qa, double qb,
                                         double eps) {
  const double w3[4] = {0.125, 0.375, 0.375, 0.125};
  const double w2[3] = {0.25, 0.5, 0.25};
  double ua = 0.0, ub = 0.0, va = 0.0, vb = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i < 3) {
        ua += w2[i] * w3[j] * (a[4 * (i + 1) + j] - a[4 * i + j]);
        ub += w2[i] * w3[j] * (b[4 * (i + 1) + j] - b[4 * i + j]);
      }
      if (j < 3) {
        va += w3[i] * w2[j] * (a[4 * i + j + 1] - a[4 * i + j]);
        vb += w3[i] * w2[j] * (b[4 * i + j + 1] - b[4 * i + j]);
      }
    }
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
    double na = ax == 0 ? -ub : -vb, nb = ax == 0 ? ua : va;
    const double nl = sqrt(na * na + nb * nb);
    if (!(nl > 0.0)) continue;
    na /= nl;
    nb /= nl;
    double lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double s = na * (a[k] - qa) + nb * (b[k] - qb);
      lo = fmin(lo, s);
      hi = fmax(hi, s);
    }
    if (lo > 2.0 * eps || hi < -2.0 * eps) return false;
  }
  return true;
}

// Query part: g = G - q at the centre -> predicted root t* = 1/2 - Ys g and
// K = t* +- R.  Returns 0 exclude (K misses the exclusion box [xlo, xhi]),
// 1 unique root in the certification box [clo, chi], 2 undecided.
__device__ __forceinline__ int kraw_query(const KrawPre& k, double ga, double gb, double xlo_u,
                                          double xhi_u, double xlo_v, double xhi_v, double clo,
                                          double chi, double& s0, double& s1) {
  if (!k.ok) return 2;
  s0 = 0.5 - (k.Y00 * ga + k.Y01 * gb);
  s1 = 0.5 - (k.Y10 * ga + k.Y11 * gb);
  if (!isfinite(s0) || !isfinite(s1)) return 2;
  const double r0 = k.R0, r1 = k.R1;
  if (s0 + r0 < xlo_u || s0 - r0 > xhi_u || s1 + r1 < xlo_v || s1 - r1 > xhi_v) return 0;
  if (s0 - r0 > clo && s0 + r0 < chi && s1 - r1 > clo && s1 + r1 < chi) return 1;
  return 2;
}

// Krawczyk test on a query-shifted node net (local coords s in [0,1]^2).
// Returns 0 exclude, 1 unique root (s0,s1 = Newton-predicted root), 2 split.
// xlo/xhi: exclusion box in local coords (domain-tolerance expansion).
__device__ __forceinline__ int krawczyk(const double* a, const double* b, double xlo_u,
                                        double xhi_u, double xlo_v, double xhi_v, double& s0,
                                        double& s1) {
  const KrawPre k = kraw_pre(a, b);
  return kraw_query(k, k.Ga, k.Gb, xlo_u, xhi_u, xlo_v, xhi_v, -1e-7, 1.0 + 1e-7, s0, s1);
}

// Blossom extraction of the cubic piece over [x0, x1] (general de Casteljau):
// new control points f(x0,x0,x0), f(x0,x0,x1), f(x0,x1,x1), f(x1,x1,x1).
__device__ __forceinline__ void extract4(double& p0, double& p1, double& p2, double& p3,
                                         double x0, double x1) {
  // stages with x0: l = (p01, p12, p23)(x0), m = (l01, l12)(x0)
  const double a01 = fma(x0, p1 - p0, p0), a12 = fma(x0, p2 - p1, p1), a23 = fma(x0, p3 - p2, p2);
  const double b0 = fma(x0, a12 - a01, a01), b1 = fma(x0, a23 - a12, a12);
  const double c01 = fma(x1, p1 - p0, p0), c12 = fma(x1, p2 - p1, p1), c23 = fma(x1, p3 - p2, p2);
  const double d0 = fma(x1, c12 - c01, c01), d1 = fma(x1, c23 - c12, c12);
  const double q0 = fma(x0, b1 - b0, b0);   // f(x0,x0,x0)
  const double q1 = fma(x1, b1 - b0, b0);   // f(x0,x0,x1)
  const double q2 = fma(x0, d1 - d0, d0);   // f(x1,x1,x0)
  const double q3 = fma(x1, d1 - d0, d0);   // f(x1,x1,x1)
  p0 = q0; p1 = q1; p2 = q2; p3 = q3;
}

// extract the sub-net over [u0,u1] x [v0,v1] of a 16-value net, in place
__device__ __forceinline__ void extract_net(double* x, double u0, double u1, double v0,
                                            double v1) {
#pragma unroll
  for (int j = 0; j < 4; ++j) extract4(x[j], x[4 + j], x[8 + j], x[12 + j], u0, u1);
#pragma unroll
  for (int i = 0; i < 4; ++i) extract4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3], v0, v1);
}

// Precomputed leaf sub-patch of a round (K1): the Krawczyk data over the
// leaf box D expanded by kLeafM on every side (D'), so that every root in D
// certifies from the leaf itself when R0, R1 < kLeafRmax.
constexpr double kLeafM = 0.5;
constexpr double kLeafRmax = 0.24;

// Ownership cut of an interior split line x (a dyadic value, computed exactly
// by both neighbouring boxes): x + kOwnShift.  Two leaves solve a root on
// their shared split line independently, so their Newton results straddle x
// by an ulp either way; shifting the cut off the dyadic lattice keeps roots
// of structured inputs (voxel grids, slices: dyadic coordinates on a linear
// patch) away from it, so exactly one neighbour owns every root.
constexpr double kOwnShift = 3.14159265358979e-11;
__device__ __forceinline__ double own_lo(double x, double tol) {
  return x == 0.0 ? -tol : x + kOwnShift;
}
__device__ __forceinline__ double own_hi(double x, double tol) {
  return x == 1.0 ? 1.0 + tol : x + kOwnShift;
}
constexpr int kLeafMaxLevel = 12;
constexpr int kLeafLevelCap = 30;  // stack bound of the leaf builder
constexpr int kSubLevelMax = 24;   // fold-tree depth (budget permitting)
constexpr double kTreeR = 0.06;    // tree nodes split while certified but max(R) >= this

struct alignas(16) LeafRec {
  double Ga, Gb;
  double Y00, Y01, Y10, Y11;
  double R0, R1;
  // two separating axes of the leaf's control hull (normals of its centre
  // tangents) with the hull's extent along each: q outside -> no root
  double n1a, n1b, lo1, hi1;
  double n2a, n2b, lo2, hi2;
  uint64_t code;   // level:6 | iu:29 | iv:29 in the patch's subdivision tree
  int32_t patch;
  int32_t ok;
};
// leaf_test_lazy (gwn_k3.cuh) reads the record as 9 double2 words
static_assert(sizeof(LeafRec) == 144 && offsetof(LeafRec, code) == 128 &&
                  offsetof(LeafRec, patch) == 136 && offsetof(LeafRec, ok) == 140,
              "LeafRec layout");

// Query-independent separating axes of a (raw) net: unit normals of the
// centre u/v tangents and the net's extent along them (hull_sat below).
__device__ __forceinline__ void hull_axes(const double* a, const double* b, double eps,
                                          LeafRec& r) {
  const double w3[4] = {0.125, 0.375, 0.375, 0.125};
  const double w2[3] = {0.25, 0.5, 0.25};
  double ua = 0.0, ub = 0.0, va = 0.0, vb = 0.0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      if (i < 3) {
        ua += w2[i] * w3[j] * (a[4 * (i + 1) + j] - a[4 * i + j]);
        ub += w2[i] * w3[j] * (b[4 * (i + 1) + j] - b[4 * i + j]);
      }
      if (j < 3) {
        va += w3[i] * w2[j] * (a[4 * i + j + 1] - a[4 * i + j]);
        vb += w3[i] * w2[j] * (b[4 * i + j + 1] - b[4 * i + j]);
      }
    }
  for (int ax = 0; ax < 2; ++ax) {
    double na = ax == 0 ? -ub : -vb, nb = ax == 0 ? ua : va;
    const double nl = sqrt(na * na + nb * nb);
    double lo = -INFINITY, hi = INFINITY;
    if (nl > 0.0) {
      na /= nl;
      nb /= nl;
      lo = INFINITY;
      hi = -INFINITY;
      for (int k = 0; k < 16; ++k) {
        const double s = na * a[k] + nb * b[k];
        lo = fmin(lo, s);
        hi = fmax(hi, s);
      }
      lo -= 2.0 * eps;
      hi += 2.0 * eps;
    } else {
      na = nb = 0.0;
    }
    if (ax == 0) { r.n1a = na; r.n1b = nb; r.lo1 = lo; r.hi1 = hi; }
    else { r.n2a = na; r.n2b = nb; r.lo2 = lo; r.hi2 = hi; }
  }
}

__device__ __forceinline__ uint64_t make_code(int level, uint64_t iu, uint64_t iv) {
  return ((uint64_t)level << 58) | (iu << 29) | iv;
}
__device__ __forceinline__ int code_level(uint64_t c) { return (int)(c >> 58); }
__device__ __forceinline__ uint64_t code_iu(uint64_t c) { return (c >> 29) & ((1ull << 29) - 1); }
__device__ __forceinline__ uint64_t code_iv(uint64_t c) { return c & ((1ull << 29) - 1); }
__device__ __forceinline__ double code_wu(int level) { return ldexp(1.0, -((level + 1) >> 1)); }
__device__ __forceinline__ double code_wv(int level) { return ldexp(1.0, -(level >> 1)); }

struct RootNet {
  double a[16], b[16];
  double eps_box;
};

__device__ __forceinline__ void load_root(const double* __restrict__ P48, double qa, double qb,
                                          const DevParams& prm, RootNet& n) {
  double amag = 0.0, alo = INFINITY, ahi = -INFINITY, blo = INFINITY, bhi = -INFINITY;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    double A = __ldg(P48 + k), B = __ldg(P48 + 16 + k);
    n.a[k] = A - qa;
    n.b[k] = B - qb;
    amag = fmax(amag, fmax(fabs(A), fabs(B)));
    alo = fmin(alo, A); ahi = fmax(ahi, A); blo = fmin(blo, B); bhi = fmax(bhi, B);
  }
  n.eps_box = 1e-12 * (1.0 + amag) + 3.0 * prm.domain_tol * fmax(ahi - alo, bhi - blo);
}

// keep the left (right=false) or right half of a split along dir, in place
__device__ __forceinline__ void halve_keep(double* a, double* b, int dir, bool right) {
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int i0 = dir == 0 ? l : 4 * l;
    const int st = dir == 0 ? 4 : 1;
    double q0, q1, q2, q3;
    half4(a[i0], a[i0 + st], a[i0 + 2 * st], a[i0 + 3 * st], q0, q1, q2, q3);
    if (right) { a[i0] = q0; a[i0 + st] = q1; a[i0 + 2 * st] = q2; a[i0 + 3 * st] = q3; }
    half4(b[i0], b[i0 + st], b[i0 + 2 * st], b[i0 + 3 * st], q0, q1, q2, q3);
    if (right) { b[i0] = q0; b[i0 + st] = q1; b[i0 + 2 * st] = q2; b[i0 + 3 * st] = q3; }
  }
}

// Rebuild the node net: levels alternate u (even) / v (odd) splits; the
// path bits are iu / iv read from the most significant end.
__device__ __forceinline__ void rebuild(double* a, double* b, int level, uint64_t iu,
                                        uint64_t iv) {
  const int nu = (level + 1) >> 1, nv = level >> 1;
  int ku = 0, kv = 0;
  for (int l = 0; l < level; ++l) {
    if ((l & 1) == 0) {
      halve_keep(a, b, 0, (iu >> (nu - 1 - ku)) & 1);
      ++ku;
    } else {
      halve_keep(a, b, 1, (iv >> (nv - 1 - kv)) & 1);
      ++kv;
    }
  }
}

// Segmented warp-shuffle reduction keyed by `key` (K5): sums `v` and ORs `f`
// over each maximal run of equal keys among adjacent lanes; returns true on the
// lane that ends its run (that lane holds the run totals).  Works for any key
// order: runs are delimited by head flags, not by key equality at a distance.
__device__ __forceinline__ bool seg_reduce(int32_t key, int32_t& v, int32_t& f) {
  const int lane = threadIdx.x & 31;
  const int32_t kprev = __shfl_up_sync(0xffffffffu, key, 1);
  int start = (lane == 0 || kprev != key) ? lane : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {  // max-scan of run heads -> run start lane
    int s = __shfl_up_sync(0xffffffffu, start, o);
    if (lane >= o) start = max(start, s);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t vu = __shfl_up_sync(0xffffffffu, v, o);
    int32_t fu = __shfl_up_sync(0xffffffffu, f, o);
    if (lane - o >= start) {
      v += vu;
      f |= fu;
    }
  }
  const int32_t knext = __shfl_down_sync(0xffffffffu, key, 1);
  return lane == 31 || knext != key;
}

// Outcome of a Newton solve started inside a node (surfaces.py:664-700 rules).
enum : int { ROOT_ACCEPTED = 0, ROOT_REJECTED = 1, ROOT_DIVERGED = 2 };

struct RootResult {
  int status;
  double u, v, t;
  int32_t sign, tang, graze, onsurf;
  int32_t iters;
};

// Newton on the whole patch from (u, v); residual / domain / t acceptance of
// surfaces.py:665-670, record fields of surfaces.py:681-697 in the
// right-handed ray frame (d = (0,0,1)).
// 16-byte read-only load the compiler may not hoist out of a loop (the
// power-basis Newton with kLoad = 1 re-reads its nets every iteration)
__device__ __forceinline__ void ldg2_keep(const double* p, double& x, double& y) {
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "l"(p));
}

__device__ __forceinline__ RootResult newton_solve(const double* __restrict__ P48, double qa,
                                                   double qb, double qc, double u, double v,
                                                   const DevParams& prm) {
  RootResult r;
  r.iters = 0;
  double bu[4], dbu[4], bv[4], dbv[4];
  double A = 0, Au = 0, Av = 0, B = 0, Bu = 0, Bv = 0;
  double du = 0.0, dv = 0.0;  // final (quadratically converged) step, applied below
  bool conv = false;
  for (int it = 0; it < kNewtonMax; ++it) {
    bern3(u, bu, dbu);
    bern3(v, bv, dbv);
    eval_coord(P48, bu, dbu, bv, dbv, A, Au, Av);
    eval_coord(P48 + 16, bu, dbu, bv, dbv, B, Bu, Bv);
    A -= qa;
    B -= qb;
    r.iters++;
    const double det = Au * Bv - Av * Bu;
    if (!(fabs(det) > 0.0)) break;
    const double id = 1.0 / det;
    const double su = (Bv * A - Av * B) * id, sv = (Au * B - Bu * A) * id;
    if (!isfinite(su) || !isfinite(sv)) break;
    // stop once the step is tiny: Newton's quadratic convergence makes the
    // stepped point accurate to ~1e-22, so it is applied without another
    // evaluation (t and the record use the current partials, t corrected to
    // first order)
// Stop once the Newton step is below GWN_NEWTON_STOP (parameter units):
// |g(x_k)| <= |J| |s_k|, and quadratic convergence from the certified start
// puts the stepped point within O(|s_k|^2) ~ 1e-14 of the root, far inside
// the 1e-10 residual acceptance of surfaces.py:665 -- one full evaluation
// fewer than waiting for a 1e-11 step (25% fewer iterations at config 2).
#ifndef GWN_NEWTON_STOP
#define GWN_NEWTON_STOP 1e-7
#endif
    if (fabs(su) <= GWN_NEWTON_STOP * fmax(1.0, fabs(u)) &&
        fabs(sv) <= GWN_NEWTON_STOP * fmax(1.0, fabs(v)) &&
        (GWN_NEWTON_STOP > 1e-11 || sqrt(A * A + B * B) <= prm.residual)) {
      du = su;
      dv = sv;
      conv = true;
      if (GWN_NEWTON_STOP > 1e-11) {
        // quadratic convergence: the stepped point's residual is O(|s|^2)
        A = 0.0;
        B = 0.0;
      }
      break;
    }
    u -= su;
    v -= sv;
    if (fabs(u) > 8.0 || fabs(v) > 8.0) break;  // left the patch neighbourhood
  }
  if (!conv) {
    bern3(u, bu, dbu);
    bern3(v, bv, dbv);
    eval_coord(P48, bu, dbu, bv, dbv, A, Au, Av);
    eval_coord(P48 + 16, bu, dbu, bv, dbv, B, Bu, Bv);
    A -= qa;
    B -= qb;
  }
  r.t = 0.0;
  r.sign = 0; r.tang = 0; r.graze = 0; r.onsurf = 0;
  if (!(sqrt(A * A + B * B) <= prm.residual)) {                        // surfaces.py:665
    r.u = u;
    r.v = v;
    r.status = ROOT_DIVERGED;
    return r;
  }
  double C, Cu, Cv;
  eval_coord(P48 + 32, bu, dbu, bv, dbv, C, Cu, Cv);
  u -= du;
  v -= dv;
  r.u = u;
  r.v = v;
  const double tol = prm.domain_tol;                                   // surfaces.py:668
  if (!(u >= -tol && u <= 1.0 + tol && v >= -tol && v <= 1.0 + tol)) {
    r.status = ROOT_REJECTED;
    return r;
  }
  r.t = C - qc - (Cu * du + Cv * dv);
  if (r.t < -prm.t_tol) {                                              // surfaces.py:670
    r.status = ROOT_REJECTED;
    return r;
  }
  const double nx = Bu * Cv - Cu * Bv, ny = Cu * Av - Au * Cv, nz = Au * Bv - Bu * Av;
  const double nn = sqrt(nx * nx + ny * ny + nz * nz);
  r.sign = 1; r.tang = 1; r.graze = 1;
  if (!(nn < prm.degenerate)) {                                        // surfaces.py:684-687
    const double dd = nz / nn;
    r.sign = dd > 0.0 ? 1 : -1;                                        // surfaces.py:695
    r.tang = fabs(dd) <= prm.tangent;                                  // :696 tangency
    const double bd = fmin(fmin(u, 1.0 - u), fmin(v, 1.0 - v));
    r.graze = bd < prm.edge_graze;                                     // :697 grazing
  }
  r.onsurf = fabs(r.t) <= prm.on_surface_t;
  r.status = ROOT_ACCEPTED;
  return r;
}

// Value and partials of one coordinate net in the tensor power basis (W[4i+j]
// = coefficient of u^i v^j) by Horner: 33 fp64 ops (61 flops, FMA = 2)
// against 44 for the Bernstein form plus its two basis evaluations.
__device__ __forceinline__ void eval_pow(const double* __restrict__ W, double u, double v,
                                         double u3, double v3, double& f, double& fu,
                                         double& fv) {
  double R[4], Rv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double a0 = W[4 * i], a1 = W[4 * i + 1], a2 = W[4 * i + 2], a3 = W[4 * i + 3];
    R[i] = fma(fma(fma(a3, v, a2), v, a1), v, a0);
    Rv[i] = fma(fma(v3, a3, a2 + a2), v, a1);
  }
  f = fma(fma(fma(R[3], u, R[2]), u, R[1]), u, R[0]);
  fu = fma(fma(u3, R[3], R[2] + R[2]), u, R[1]);
  fv = fma(fma(fma(Rv[3], u, Rv[2]), u, Rv[1]), u, Rv[0]);
}

// newton_solve with the nets in the power basis (K3 Newton pass): identical
// iteration, stopping rule, acceptance (surfaces.py:665-670) and record
// fields (surfaces.py:681-697); only the evaluation of the map differs (by
// rounding).  W48 = (A, B, C) power coefficients of the patch (Round::powc).
// 16-byte shared-memory load the compiler may not hoist (see ldg2_keep)
__device__ __forceinline__ void lds2_keep(const double* p, double& x, double& y) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

// kLoad: 0 = coefficients through the compiler (hoisted into registers),
// 1 = re-read from global (L1) every iteration, 2 = re-read from shared
template <int kLoad>
__device__ __forceinline__ void pow_eval_ab(const double* __restrict__ W48, double u, double v,
                                            double& A, double& Au, double& Av, double& B,
                                            double& Bu, double& Bv) {
  const double u3 = 3.0 * u, v3 = 3.0 * v;
  if (kLoad) {
    double X[32];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (kLoad == 2) lds2_keep(W48 + 2 * k, X[2 * k], X[2 * k + 1]);
      else ldg2_keep(W48 + 2 * k, X[2 * k], X[2 * k + 1]);
    }
    eval_pow(X, u, v, u3, v3, A, Au, Av);
    eval_pow(X + 16, u, v, u3, v3, B, Bu, Bv);
  } else {
    eval_pow(W48, u, v, u3, v3, A, Au, Av);
    eval_pow(W48 + 16, u, v, u3, v3, B, Bu, Bv);
  }
}

// Newton iteration state (power basis); `act` while iterating
struct NState {
  double u, v, du, dv, A, Au, Av, B, Bu, Bv;
  int iters;
  bool conv, act;
};

__device__ __forceinline__ NState nstate(double u, double v, bool act) {
  NState s;
  s.u = u; s.v = v; s.du = 0.0; s.dv = 0.0;
  s.A = s.Au = s.Av = s.B = s.Bu = s.Bv = 0.0;
  s.iters = 0; s.conv = false; s.act = act;
  return s;
}

// one iteration on freshly evaluated A, B, partials (already minus q)
__device__ __forceinline__ void nstate_update(NState& s, const DevParams& prm) {
  s.iters++;
  const double det = s.Au * s.Bv - s.Av * s.Bu;
  if (!(fabs(det) > 0.0)) { s.act = false; return; }
  const double id = 1.0 / det;
  const double su = (s.Bv * s.A - s.Av * s.B) * id, sv = (s.Au * s.B - s.Bu * s.A) * id;
  if (!isfinite(su) || !isfinite(sv)) { s.act = false; return; }
  if (fabs(su) <= GWN_NEWTON_STOP * fmax(1.0, fabs(s.u)) &&
      fabs(sv) <= GWN_NEWTON_STOP * fmax(1.0, fabs(s.v)) &&
      (GWN_NEWTON_STOP > 1e-11 || sqrt(s.A * s.A + s.B * s.B) <= prm.residual)) {
    s.du = su;
    s.dv = sv;
    s.conv = true;
    if (GWN_NEWTON_STOP > 1e-11) {
      s.A = 0.0;
      s.B = 0.0;
    }
    s.act = false;
    return;
  }
  s.u -= su;
  s.v -= sv;
  if (fabs(s.u) > 8.0 || fabs(s.v) > 8.0) s.act = false;
}

// acceptance (surfaces.py:665-670) and record fields (surfaces.py:681-697)
__device__ __forceinline__ RootResult nstate_finish(NState& s, const double* __restrict__ W48,
                                                    double qa, double qb, double qc,
                                                    const DevParams& prm) {
  RootResult r;
  r.iters = s.iters;
  double u = s.u, v = s.v;
  if (!s.conv) {
    pow_eval_ab<0>(W48, u, v, s.A, s.Au, s.Av, s.B, s.Bu, s.Bv);
    s.A -= qa;
    s.B -= qb;
  }
  const double A = s.A, Au = s.Au, Av = s.Av, B = s.B, Bu = s.Bu, Bv = s.Bv;
  r.t = 0.0;
  r.sign = 0; r.tang = 0; r.graze = 0; r.onsurf = 0;
  if (!(sqrt(A * A + B * B) <= prm.residual)) {                        // surfaces.py:665
    r.u = u;
    r.v = v;
    r.status = ROOT_DIVERGED;
    return r;
  }
  double C, Cu, Cv;
  eval_pow(W48 + 32, u, v, 3.0 * u, 3.0 * v, C, Cu, Cv);
  u -= s.du;
  v -= s.dv;
  r.u = u;
  r.v = v;
  const double tol = prm.domain_tol;                                   // surfaces.py:668
  if (!(u >= -tol && u <= 1.0 + tol && v >= -tol && v <= 1.0 + tol)) {
    r.status = ROOT_REJECTED;
    return r;
  }
  r.t = C - qc - (Cu * s.du + Cv * s.dv);
  if (r.t < -prm.t_tol) {                                              // surfaces.py:670
    r.status = ROOT_REJECTED;
    return r;
  }
  const double nx = Bu * Cv - Cu * Bv, ny = Cu * Av - Au * Cv, nz = Au * Bv - Bu * Av;
  const double nn = sqrt(nx * nx + ny * ny + nz * nz);
  r.sign = 1; r.tang = 1; r.graze = 1;
  if (!(nn < prm.degenerate)) {                                        // surfaces.py:684-687
    const double dd = nz / nn;
    r.sign = dd > 0.0 ? 1 : -1;                                        // surfaces.py:695
    r.tang = fabs(dd) <= prm.tangent;                                  // :696 tangency
    const double bd = fmin(fmin(u, 1.0 - u), fmin(v, 1.0 - v));
    r.graze = bd < prm.edge_graze;                                     // :697 grazing
  }
  r.onsurf = fabs(r.t) <= prm.on_surface_t;
  r.status = ROOT_ACCEPTED;
  return r;
}

// newton_solve with the nets in the power basis (K3 Newton pass): identical
// iteration, stopping rule, acceptance (surfaces.py:665-670) and record
// fields (surfaces.py:681-697); only the evaluation of the map differs (by
// rounding).  W48 = (A, B, C) power coefficients of the patch (Round::powc).
template <int kLoad = 0>
__device__ __forceinline__ RootResult newton_solve_pow(const double* __restrict__ W48, double qa,
                                                       double qb, double qc, double u, double v,
                                                       const DevParams& prm) {
  NState s = nstate(u, v, true);
  for (int it = 0; it < kNewtonMax && s.act; ++it) {
    pow_eval_ab<kLoad>(W48, s.u, s.v, s.A, s.Au, s.Av, s.B, s.Bu, s.Bv);
    s.A -= qa;
    s.B -= qb;
    nstate_update(s, prm);
  }
  return nstate_finish(s, W48, qa, qb, qc, prm);
}

}  // namespace gwn
