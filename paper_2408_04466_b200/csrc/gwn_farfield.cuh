// gwn_farfield.cuh -- far field of the boundary term.
//
// The net boundary is the boundary of a surface, so every connected component
// of its edge graph is a closed cycle.  For a closed cycle, K4's fan sum from
// c = -d equals the cycle's solid angle Omega(p) (the fan-from-centre surface)
// whenever the line p + t d misses the cycle's bounding sphere: no 4 pi branch
// and no band re-shoot.  Outside the sphere Omega is harmonic and has the
// multipole expansion
//     Omega(p) = -sum_{n>=1} sum_{m=-n..n} D_n^m I_n^m(p - g),
//     D_n^m = integral over the fan surface of n . conj(grad R_n^m(x - g)) dA,
// with the regular / irregular solid harmonics R, I of the addition theorem
// 1/|p - q| = sum_n sum_m conj(R_n^m(q)) I_n^m(p) (recurrences in
// gwn_farfield.cu; checked in tools/farfield/proto.py).  Keeping n <= K keeps
// the degree-(K-1) part of grad_q 1/|p-q| in delta = q - g; the dropped part
// is bounded two ways (ff_bound takes the smaller):
//   Taylor remainder with |d^k (1/r)| <= k!/r^(k+1) along unit directions:
//     A_abs (K+1) rho^K / (R - rho)^(K+2);
//   Legendre tail: grad of |d|^n P_n(cos) is <= sqrt(2) n |d|^(n-1) (|P_n| <= 1
//   and Bernstein's inequality), summed over n > K:
//     sqrt(2) A_abs (K+1) rho^K / (R^K (R - rho)^2).
// A (query, cycle) pair is "far" when R^2 >= R_min^2 with the bound at the
// scene's tau and either the forward half-line misses the sphere or its
// shadow cell is clean (gwn_boundary.cu, ff_class).  Every K4 pass takes the
// decision with ff_class on the same bits, so the exact and far pairs
// partition the (query, cycle) pairs exactly.
#pragma once

#include <math.h>

#include "gwn_internal.h"

namespace gwn {

// Largest expansion order of the per-pair path.  R_min, the radius inside
// which a pair takes the exact sum, comes from the order-K a-priori bound:
// ~4.3 cycle radii at order 20, ~2.2 at 48, ~1.9 at 64.  Pairs farther out
// use the lowest sufficient order (kFFLevels).  Measured at config 5, 2^23
// queries (tools/farfield/order_ab.py): K = 48: 8.53 M near pairs, eval
// 46.6 ms; 56: 7.00 M, 43.7 ms; 64: 6.05 M, 42.9 ms (the far pairs gained
// cost 2.2 ms, the near pairs lost save 6.2 ms; the moments of a scene take
// ~1 s longer to integrate).
#ifndef GWN_FF_K
#define GWN_FF_K 64
#endif
constexpr int kFFK = GWN_FF_K;
constexpr int kFFTerms = (kFFK + 1) * (kFFK + 2) / 2;  // (n, m), 0 <= m <= n <= K
// Error budget of the far field: every expanded entry's truncation is bounded
// by tau = 2 pi kFFDw / (expanded entries) (Omega units, per pair; the FMM
// splits it into two halves), so the far field moves a query's w by at most
// kFFDw -- two orders below the north star's 1e-6.  The lower orders'
// thresholds come from the computed moments (gwn_farfield.cu), a tight bound:
// measured differences from the exact sum reach 2e-12 (config 5) and 4e-11
// (config 3); with the a-priori bound alone they stayed near 1e-14.
constexpr double kFFDw = 1e-8;
// far-field partial rows: cycle groups summed in fixed order by K5, so the
// far kernel fills the GPU and w stays bit-identical for any batching
constexpr int kFFRows = 16;
// adaptive order: a far pair uses the lowest of these orders whose bound
// holds at its distance (per-cycle thresholds, Scene::ff_lv)
constexpr int kFFLevels = (kFFK - 12) / 4 + 1;  // orders 12, 16, ..., kFFK
__host__ __device__ constexpr int ff_order(int lv) { return kFFK - 4 * (kFFLevels - 1 - lv); }

__host__ __device__ __forceinline__ constexpr int ff_term(int n, int m) {
  return n * (n + 1) / 2 + m;
}

// local expansions (gwn_fmm.cu): order of the leaves' expansions, their
// (j, k >= 0) coefficient count, the irregular-harmonic degree M2L needs
// order of the leaves' local expansions.  Measured at config 5, 2^23 queries
// (tools/farfield/order_ab.py): P = 20: 48.8 M per-pair far pairs, eval
// 42.6 ms; 24: 43.6 M, 41.7 ms; 28: 42.2 M, 46.3 ms (the L2P grows faster than
// the leftover pairs shrink).
#ifndef GWN_FMM_P
#define GWN_FMM_P 24
#endif
constexpr int kFmmP = GWN_FMM_P;
constexpr int kFmmK = 30;  // multipole order translated by M2L (<= kFFK)
constexpr int kFmmLT = (kFmmP + 1) * (kFmmP + 2) / 2;
constexpr int kFmmKT = (kFmmK + 1) * (kFmmK + 2) / 2;
constexpr int kFmmIN = kFmmK + kFmmP;
constexpr int kFmmIT = (kFmmIN + 1) * (kFmmIN + 2) / 2;

// Omega(z + x) = sum_j [Re(conj(R_j^0(x)) L_j^0) + 2 sum_{k>=1} Re(conj(R_j^k(x)) L_j^k)]
// (L2P), the regular harmonics by the recurrences of gwn_farfield.cu's
// moment kernel: R_0^0 = 1, R_m^m = -(x+iy)/(2m) R_{m-1}^{m-1},
// R_n^m = ((2n-1) z R_{n-1}^m - r^2 R_{n-2}^m) / ((n+m)(n-m)).
__device__ __forceinline__ double fmm_l2p(double x, double y, double z,
                                          const double2* __restrict__ Lc) {
  const double r2 = x * x + y * y + z * z;
  double dR = 1.0, dI = 0.0, acc = 0.0;
#pragma unroll
  for (int m = 0; m <= kFmmP; ++m) {
    if (m > 0) {
      const double c0 = -1.0 / (2.0 * m);
      const double nR = c0 * (x * dR - y * dI), nI = c0 * (x * dI + y * dR);
      dR = nR;
      dI = nI;
    }
    double aR = dR, aI = dI, bR = 0.0, bI = 0.0, col = 0.0;
#pragma unroll
    for (int n = m; n <= kFmmP; ++n) {
      if (n > m) {
        const double inv = 1.0 / ((double)(n + m) * (double)(n - m));
        const double k1 = (2.0 * n - 1.0) * z;
        const double vR = (k1 * aR - r2 * bR) * inv, vI = (k1 * aI - r2 * bI) * inv;
        bR = aR;
        bI = aI;
        aR = vR;
        aI = vI;
      }
      const double2 l = Lc[ff_term(n, m)];
      col = fma(aR, l.x, fma(aI, l.y, col));  // Re(conj(R) L)
    }
    acc += m == 0 ? col : 2.0 * col;
  }
  return acc;
}

// truncation bound of the order-K expansion at distance R (see above; host)
inline double ff_bound(double aabs, double rho, int K, double R) {
  if (!(R > rho)) return INFINITY;
  const double x = rho / R;
  const double taylor = aabs * (K + 1.0) * pow(rho, (double)K) / pow(R - rho, K + 2.0);
  const double legendre = 1.4142135623730951 * aabs * (K + 1.0) * pow(x, (double)K) /
                          ((R - rho) * (R - rho));
  return fmin(taylor, legendre);
}

// query in the round frame (explicit roundings: every kernel that takes a
// far-field decision computes bit-identical coordinates)
__device__ __forceinline__ void frame_q(const Frame& f, double px, double py, double pz,
                                        double& qa, double& qb, double& qc) {
  qa = __fma_rn(pz, f.e1[2], __fma_rn(py, f.e1[1], __dmul_rn(px, f.e1[0])));
  qb = __fma_rn(pz, f.e2[2], __fma_rn(py, f.e2[1], __dmul_rn(px, f.e2[0])));
  qc = __fma_rn(pz, f.d[2], __fma_rn(py, f.d[1], __dmul_rn(px, f.d[0])));
}

}  // namespace gwn
