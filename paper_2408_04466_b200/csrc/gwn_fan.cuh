// gwn_fan.cuh -- angle-sum helpers shared by the boundary term (K4,
// gwn_boundary.cu) and the mesh solid-angle kernel (gwn_mesh.cu): a running
// complex product Z *= (den + i num) with an exact branch-cut counter, so a
// sum of atan2(num, den) costs one atan2 per query, and a full-precision
// reciprocal square root.
#pragma once

#include "gwn_internal.h"

namespace gwn {

struct SegState {
  double Zr, Zi;
  int wraps;
};

__device__ __forceinline__ bool signbit_hi(double x) { return __double2hiint(x) < 0; }

// multiply Z by (den + i num) with exact branch-cut bookkeeping
__device__ __forceinline__ void cmul_track(SegState& s, double den, double num) {
  const double zr = s.Zr * den - s.Zi * num;
  const double zi = s.Zr * num + s.Zi * den;
  // arg(Z) + arg(z) crossed +pi (both upper half-planes, result lower) or
  // -pi (both lower, result upper); sign bits of the high words
  const unsigned a = (unsigned)__double2hiint(s.Zi), b = (unsigned)__double2hiint(num),
                 c = (unsigned)__double2hiint(zi);
  s.wraps += (int)((~a & ~b & c) >> 31) - (int)((a & b & ~c) >> 31);
  s.Zr = zr;
  s.Zi = zi;
}

__device__ __forceinline__ void renorm(SegState& s) {
  double m = fmax(fabs(s.Zr), fabs(s.Zi));
  int e = ((__double2hiint(m) >> 20) & 0x7ff);
  if (e == 0 || e == 0x7ff) return;  // zero/denormal/non-finite: degenerate, flagged elsewhere
  double sc = __hiloint2double((2046 - e) << 20, 0);  // 2^(1023-e), exact
  s.Zr *= sc;
  s.Zi *= sc;
}

// Full-precision reciprocal square root: MUFU.RSQ64H seed (~2^-22) + one
// Halley step y(1 + e/2 + 3e^2/8), e = 1 - x y^2 (cubic convergence); no
// special-value path (x > 0 unless the query sits on a vertex, which the
// degenerate test flags).  Accuracy checked by gwn_selftest_rsqrt.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = x * y;
  const double e = fma(-h, y, 1.0);
  const double p = fma(0.375, e, 0.5);
  return fma(y * e, p, y);
}

// sum of the atan2 arguments accumulated in s
__device__ __forceinline__ double seg_angle(const SegState& s) {
  return atan2(s.Zi, s.Zr) + 6.283185307179586476925 * (double)s.wraps;
}

}  // namespace gwn
