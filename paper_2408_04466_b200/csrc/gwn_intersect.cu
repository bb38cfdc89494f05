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
#include "gwn_internal.h"

namespace gwn {

constexpr int kMaxLevel = 44;
constexpr int kNodeBudget = 4096;
constexpr int kMaxRoots = 8;
constexpr int kStackNets = 24;
constexpr int kNewtonMax = 16;

struct PairOut {
  int32_t chi;
  int32_t flags;
  int32_t nodes;
  int32_t newton;
  int32_t roots;
};

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

// Krawczyk test on the node net (local coords s in [0,1]^2).
// Returns 0 exclude, 1 unique root (s0,s1 = Newton-predicted root), 2 split.
// xlo/xhi: exclusion box in local coords (domain-tolerance expansion).
__device__ __forceinline__ int krawczyk(const double* a, const double* b, double xlo_u,
                                        double xhi_u, double xlo_v, double xhi_v, double& s0,
                                        double& s1) {
  const double w3[4] = {0.125, 0.375, 0.375, 0.125};
  const double w2[3] = {0.25, 0.5, 0.25};
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
  // derivative nets are 3 x differences; fold the 3 into Y
  double det = Jua * Jvb - Jva * Jub;
  if (!(fabs(det) > 1e-300) || !isfinite(det)) return 2;
  double id = 1.0 / det;
  double Y00 = Jvb * id, Y01 = -Jva * id, Y10 = -Jub * id, Y11 = Jua * id;  // (J/3)^-1
  double d0 = (Y00 * ga + Y01 * gb) * (1.0 / 3.0);
  double d1 = (Y10 * ga + Y11 * gb) * (1.0 / 3.0);
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
  double r0 = (e11 + e12) * rad * (1.0 + 1e-9) + 1e-12;
  double r1 = (e21 + e22) * rad * (1.0 + 1e-9) + 1e-12;
  s0 = 0.5 - d0;
  s1 = 0.5 - d1;
  if (!isfinite(s0) || !isfinite(s1)) return 2;
  if (s0 + r0 < xlo_u || s0 - r0 > xhi_u || s1 + r1 < xlo_v || s1 - r1 > xhi_v) return 0;
  if (s0 - r0 > -1e-7 && s0 + r0 < 1.0 + 1e-7 && s1 - r1 > -1e-7 && s1 + r1 < 1.0 + 1e-7)
    return 1;
  return 2;
}

template <bool kRecord>
struct RootAcc {
  double t[kMaxRoots];
  int n;
  int32_t chi;
  int32_t flags;
  int32_t newton;
};

template <>
struct RootAcc<true> {
  double t[kMaxRoots], u[kMaxRoots], v[kMaxRoots];
  int32_t sign[kMaxRoots], tang[kMaxRoots], graze[kMaxRoots];
  int n;
  int32_t chi;
  int32_t flags;
  int32_t newton;
};

// Newton on the whole patch from (u,v); on acceptance record the root.
template <bool kRecord>
__device__ void newton_root(const double* __restrict__ P48, double qa, double qb, double qc,
                            double u, double v, const DevParams& prm, RootAcc<kRecord>& acc) {
  double bu[4], dbu[4], bv[4], dbv[4];
  double A, Au, Av, B, Bu, Bv;
  bool conv = false;
  for (int it = 0; it < kNewtonMax; ++it) {
    bern3(u, bu, dbu);
    bern3(v, bv, dbv);
    eval_coord(P48, bu, dbu, bv, dbv, A, Au, Av);
    eval_coord(P48 + 16, bu, dbu, bv, dbv, B, Bu, Bv);
    A -= qa;
    B -= qb;
    acc.newton++;
    double det = Au * Bv - Av * Bu;
    if (!(fabs(det) > 0.0)) break;
    double id = 1.0 / det;
    double du = (Bv * A - Av * B) * id, dv = (Au * B - Bu * A) * id;
    if (!isfinite(du) || !isfinite(dv)) break;
    if (fabs(du) <= 2e-16 * fmax(1.0, fabs(u)) && fabs(dv) <= 2e-16 * fmax(1.0, fabs(v))) {
      conv = true;
      break;
    }
    u -= du;
    v -= dv;
    if (fabs(u) > 8.0 || fabs(v) > 8.0) break;  // left the patch neighbourhood
  }
  if (!conv) {
    // final evaluation at the last iterate (xtol-style stop, surfaces.py:662)
    bern3(u, bu, dbu);
    bern3(v, bv, dbv);
    eval_coord(P48, bu, dbu, bv, dbv, A, Au, Av);
    eval_coord(P48 + 16, bu, dbu, bv, dbv, B, Bu, Bv);
    A -= qa;
    B -= qb;
  }
  if (!(sqrt(A * A + B * B) <= prm.residual)) return;                 // surfaces.py:665
  const double tol = prm.domain_tol;                                  // surfaces.py:668
  if (!(u >= -tol && u <= 1.0 + tol && v >= -tol && v <= 1.0 + tol)) return;
  double C, Cu, Cv;
  eval_coord(P48 + 32, bu, dbu, bv, dbv, C, Cu, Cv);
  double t = C - qc;
  if (t < -prm.t_tol) return;                                         // surfaces.py:670
  for (int k = 0; k < acc.n; ++k)                                     // surfaces.py:672-674
    if (fabs(acc.t[k] - t) < prm.dedup) return;
  if (acc.n >= kMaxRoots) {
    acc.flags |= FLAG_RESHOOT;
    return;
  }
  const int k = acc.n++;
  acc.t[k] = t;
  // record (surfaces.py:681-697) in the right-handed ray frame: d = (0,0,1)
  double nx = Bu * Cv - Cu * Bv, ny = Cu * Av - Au * Cv, nz = Au * Bv - Bu * Av;
  double nn = sqrt(nx * nx + ny * ny + nz * nz);
  int32_t sign = 1, tang = 1, graze = 1;
  if (!(nn < prm.degenerate)) {                                       // surfaces.py:684-687
    double dd = nz / nn;
    sign = dd > 0.0 ? 1 : -1;                                         // surfaces.py:695
    tang = fabs(dd) <= prm.tangent;                                   // :696 tangency
    double bd = fmin(fmin(u, 1.0 - u), fmin(v, 1.0 - v));
    graze = bd < prm.edge_graze;                                      // :697 grazing
  }
  acc.chi += sign;
  if (tang || graze) acc.flags |= FLAG_RESHOOT;
  if (fabs(t) <= prm.on_surface_t) acc.flags |= FLAG_ONSURF;
  if constexpr (kRecord) {
    acc.u[k] = u;
    acc.v[k] = v;
    acc.sign[k] = sign;
    acc.tang[k] = tang;
    acc.graze[k] = graze;
  }
}

// Complete root enumeration for one (query, patch) pair.
template <bool kRecord>
__device__ PairOut solve_pair(const double* __restrict__ P48, double qa, double qb, double qc,
                              const DevParams& prm, RootAcc<kRecord>& acc) {
  double a[16], b[16];
  double amag = 0.0, alo = INFINITY, ahi = -INFINITY, blo = INFINITY, bhi = -INFINITY;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    double A = __ldg(P48 + k), B = __ldg(P48 + 16 + k);
    a[k] = A - qa;
    b[k] = B - qb;
    amag = fmax(amag, fmax(fabs(A), fabs(B)));
    alo = fmin(alo, A); ahi = fmax(ahi, A); blo = fmin(blo, B); bhi = fmax(bhi, B);
  }
  const double eps_box = 1e-12 * (1.0 + amag) + 3.0 * prm.domain_tol * fmax(ahi - alo, bhi - blo);
  acc.n = 0;
  acc.chi = 0;
  acc.flags = 0;
  acc.newton = 0;
  int nodes = 0;
  double st_a[kStackNets][16], st_b[kStackNets][16];
  double st_box[kStackNets][3];  // u0, v0, level
  int top = 0;
  double u0 = 0.0, v0 = 0.0;
  int level = 0;
  bool have = box_has_origin(a, b, eps_box);
  while (have) {
    ++nodes;
    if (nodes > kNodeBudget) {
      acc.flags |= FLAG_RESHOOT;
      break;
    }
    // node widths: levels alternate u, v splits (u first)
    double wu = ldexp(1.0, -((level + 1) >> 1));
    double wv = ldexp(1.0, -(level >> 1));
    double xlo_u = u0 == 0.0 ? -prm.domain_tol / wu : 0.0;
    double xhi_u = u0 + wu == 1.0 ? 1.0 + prm.domain_tol / wu : 1.0;
    double xlo_v = v0 == 0.0 ? -prm.domain_tol / wv : 0.0;
    double xhi_v = v0 + wv == 1.0 ? 1.0 + prm.domain_tol / wv : 1.0;
    double s0, s1;
    int kr = krawczyk(a, b, xlo_u, xhi_u, xlo_v, xhi_v, s0, s1);
    bool pop = true;
    if (kr == 1) {
      newton_root(P48, qa, qb, qc, u0 + s0 * wu, v0 + s1 * wv, prm, acc);
    } else if (kr == 2) {
      if (level >= kMaxLevel) {
        newton_root(P48, qa, qb, qc, u0 + 0.5 * wu, v0 + 0.5 * wv, prm, acc);
      } else {
        int dir = (level & 1);  // 0: split u, 1: split v
        double ra[16], rb[16];
        split_net(a, b, ra, rb, dir);
        double ru0 = dir == 0 ? u0 + 0.5 * wu : u0;
        double rv0 = dir == 1 ? v0 + 0.5 * wv : v0;
        ++level;
        bool okL = box_has_origin(a, b, eps_box);
        bool okR = box_has_origin(ra, rb, eps_box);
        if (okL && okR) {
          if (top < kStackNets) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              st_a[top][k] = ra[k];
              st_b[top][k] = rb[k];
            }
            st_box[top][0] = ru0;
            st_box[top][1] = rv0;
            st_box[top][2] = (double)level;
            ++top;
          } else {
            acc.flags |= FLAG_RESHOOT;
          }
          pop = false;
        } else if (okL) {
          pop = false;
        } else if (okR) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            a[k] = ra[k];
            b[k] = rb[k];
          }
          u0 = ru0;
          v0 = rv0;
          pop = false;
        }
      }
    }
    if (pop) {
      if (top == 0) break;
      --top;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        a[k] = st_a[top][k];
        b[k] = st_b[top][k];
      }
      u0 = st_box[top][0];
      v0 = st_box[top][1];
      level = (int)st_box[top][2];
    }
  }
  PairOut o;
  o.chi = acc.chi;
  o.flags = acc.flags;
  o.nodes = nodes;
  o.newton = acc.newton;
  o.roots = acc.n;
  return o;
}

__device__ __forceinline__ void warp_add_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

__global__ void __launch_bounds__(128)
k_intersect(int64_t npairs, const int32_t* __restrict__ pair_slot,
            const int32_t* __restrict__ pair_patch, const double* __restrict__ qproj,
            const double* __restrict__ proj, DevParams prm, int32_t* __restrict__ chi_acc,
            int32_t* __restrict__ flag_acc, unsigned long long* __restrict__ counters) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t slot = -1;
  PairOut r = {0, 0, 0, 0, 0};
  if (i < npairs) {
    slot = pair_slot[i];
    int32_t p = pair_patch[i];
    double qa = qproj[3 * (int64_t)slot], qb = qproj[3 * (int64_t)slot + 1],
           qc = qproj[3 * (int64_t)slot + 2];
    RootAcc<false> acc;
    r = solve_pair(proj + 48 * (int64_t)p, qa, qb, qc, prm, acc);
  }
  __syncwarp();
  // K5 part 1: segmented warp-shuffle reduction of (chi, flags) keyed by the
  // query slot (pairs are grouped by slot), one atomic per segment.
  const int lane = threadIdx.x & 31;
  int32_t chi = r.chi, fl = r.flags;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t s_up = __shfl_up_sync(0xffffffffu, slot, o);
    int32_t c_up = __shfl_up_sync(0xffffffffu, chi, o);
    int32_t f_up = __shfl_up_sync(0xffffffffu, fl, o);
    if (lane >= o && s_up == slot) {
      chi += c_up;
      fl |= f_up;
    }
  }
  int32_t s_next = __shfl_down_sync(0xffffffffu, slot, 1);
  bool tail = (lane == 31) || (s_next != slot);
  if (slot >= 0 && tail) {
    if (chi) atomicAdd(&chi_acc[slot], chi);
    if (fl) atomicOr(&flag_acc[slot], fl);
  }
  warp_add_u64(&counters[CNT_NODES], (unsigned long long)r.nodes);
  warp_add_u64(&counters[CNT_NEWTON], (unsigned long long)r.newton);
  warp_add_u64(&counters[CNT_ROOTS], (unsigned long long)r.roots);
}

cudaError_t launch_intersect(const gwn_scene* sc, const Round& rd, int64_t npairs,
                             const int32_t* pair_slot, const int32_t* pair_patch,
                             const double* qproj, int32_t* chi, int32_t* flags,
                             unsigned long long* counters, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  int64_t blocks = (npairs + 127) / 128;
  k_intersect<<<(unsigned)blocks, 128, 0, st>>>(npairs, pair_slot, pair_patch, qproj, rd.proj,
                                                 sc->dprm, chi, flags, counters);
  return cudaGetLastError();
}

// patch.all_hits(ray) for one ray and one patch (host API, surfaces.py:587-589):
// out rows = (t, u, v, sign, tangency, grazing), sorted by t (surfaces.py:700).
__global__ void k_all_hits(const double* __restrict__ P48, Frame f, double ox, double oy,
                           double oz, DevParams prm, double* __restrict__ out,
                           int32_t* __restrict__ count, int32_t cap) {
  double qa = ox * f.e1[0] + oy * f.e1[1] + oz * f.e1[2];
  double qb = ox * f.e2[0] + oy * f.e2[1] + oz * f.e2[2];
  double qc = ox * f.d[0] + oy * f.d[1] + oz * f.d[2];
  RootAcc<true> acc;
  solve_pair(P48, qa, qb, qc, prm, acc);
  // insertion sort by t
  int idx[kMaxRoots];
  for (int k = 0; k < acc.n; ++k) idx[k] = k;
  for (int i = 1; i < acc.n; ++i) {
    int key = idx[i], j = i - 1;
    while (j >= 0 && acc.t[idx[j]] > acc.t[key]) { idx[j + 1] = idx[j]; --j; }
    idx[j + 1] = key;
  }
  for (int k = 0; k < acc.n && k < cap; ++k) {
    int q = idx[k];
    double* row = out + 6 * k;
    row[0] = acc.t[q]; row[1] = acc.u[q]; row[2] = acc.v[q];
    row[3] = acc.sign[q]; row[4] = acc.tang[q]; row[5] = acc.graze[q];
  }
  *count = (acc.flags & FLAG_RESHOOT) && acc.n == 0 ? 0 : acc.n;
}

cudaError_t launch_all_hits(const gwn_scene* sc, const Round& rd, int64_t patch,
                            const double* o, double* out, int32_t* count, int32_t cap,
                            cudaStream_t st) {
  k_all_hits<<<1, 1, 0, st>>>(rd.proj + 48 * patch, rd.f, o[0], o[1], o[2], sc->dprm, out, count,
                              cap);
  return cudaGetLastError();
}

}  // namespace gwn
