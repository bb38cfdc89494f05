// gwn_intersect.cu -- K3: ray x bicubic-patch all-roots intersection in fp64.
//
// Replaces _multistart_ray_roots (surfaces.py:634-701): the reference seeds
// scipy root(hybr) at the domain centre with t seeds only (:645-660) and
// misses roots.  Here every (query, patch) candidate pair is
// solved completely in the ray frame (e1, e2, d) of the round: the root set
// of g(u,v) = (A(u,v) - p.e1, B(u,v) - p.e2) = 0 is enumerated by a
// depth-first subdivision of the projected 2-D control net.  Each node is
//   1. dropped if the origin is outside its control-point box (convex hull),
//   2. tested with the Krawczyk operator
//        K = c - Y g(c) + (I - Y J(D)) (D - c),  Y = J(c)^-1,
//      where J(D) is bounded by the Bernstein hulls of the derivative nets:
//      K cap D = {} -> no root; K inside D -> exactly one root, found by
//      Newton; otherwise split (de Casteljau at 1/2 along the wider side).
// Accepted roots obey the reference's rules (surfaces.py:664-700): residual
// <= 1e-10, (u,v) in the domain +-1e-9, t >= -1e-12, 1e-9 dedup, sign from
// d.n with n = f_u x f_v, tangency |d.n^| <= 1e-12, grazing if the domain
// boundary distance < 1e-10.  Per-pair chi and flags are combined per query
// with a segmented warp-shuffle reduction (K5) before one atomic per segment.
#include "gwn_dfs.cuh"

namespace gwn {

// patch.all_hits(ray, t_window, eps) for one ray and one patch (host API,
// surfaces.py:587-589): out rows = (t, u, v, sign, tangency, grazing) of the
// roots inside the t window (+-1e-12, surfaces.py:679), sorted by t
// (surfaces.py:700).  *count = number of such roots (rows past `cap` are not
// written); *flags = the root set's flag bits (FLAG_RESHOOT for tangent /
// grazing / undecided contacts).
__global__ void k_all_hits(const double* __restrict__ P48, Frame f, double ox, double oy,
                           double oz, DevParams prm, double t_lo, double t_hi,
                           double* __restrict__ out, int32_t* __restrict__ count, int32_t cap) {
  double qa = ox * f.e1[0] + oy * f.e1[1] + oz * f.e1[2];
  double qb = ox * f.e2[0] + oy * f.e2[1] + oz * f.e2[2];
  double qc = ox * f.d[0] + oy * f.d[1] + oz * f.d[2];
  RootAcc<true> acc;
  solve_pair(P48, qa, qb, qc, prm, 0, kMaxLevel, acc);
  // insertion sort by t
  int idx[kMaxRoots];
  for (int k = 0; k < acc.n; ++k) idx[k] = k;
  for (int i = 1; i < acc.n; ++i) {
    int key = idx[i], j = i - 1;
    while (j >= 0 && acc.t[idx[j]] > acc.t[key]) { idx[j + 1] = idx[j]; --j; }
    idx[j + 1] = key;
  }
  int m = 0;
  for (int k = 0; k < acc.n; ++k) {
    const int q = idx[k];
    if (acc.t[q] < t_lo - 1e-12 || acc.t[q] > t_hi + 1e-12) continue;  // surfaces.py:679
    if (m < cap) {
      double* row = out + 6 * m;
      row[0] = acc.t[q]; row[1] = acc.u[q]; row[2] = acc.v[q];
      row[3] = acc.sign[q]; row[4] = acc.tang[q]; row[5] = acc.graze[q];
    }
    ++m;
  }
  count[0] = m;
  count[1] = acc.flags;
}

cudaError_t launch_all_hits(const Round& rd, const DevParams& prm, const double* o, double t_lo,
                            double t_hi, double* out, int32_t* count, int32_t cap,
                            cudaStream_t st) {
  k_all_hits<<<1, 1, 0, st>>>(rd.proj, rd.f, o[0], o[1], o[2], prm, t_lo, t_hi, out, count,
                              cap);
  return cudaGetLastError();
}

}  // namespace gwn
