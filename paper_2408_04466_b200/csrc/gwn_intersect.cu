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
#include "gwn_patch.cuh"

namespace gwn {

constexpr int kMaxRoots = 8;
constexpr int kStackNets = 24;

struct PairOut {
  int32_t chi;
  int32_t flags;
  int32_t nodes;
  int32_t newton;
  int32_t roots;
};

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

// Newton on the whole patch from (u,v); on acceptance record the root with
// the reference's 1e-9 dedup (surfaces.py:672-674).
template <bool kRecord>
__device__ void newton_root(const double* __restrict__ P48, double qa, double qb, double qc,
                            double u, double v, const DevParams& prm, RootAcc<kRecord>& acc) {
  RootResult r = newton_solve(P48, qa, qb, qc, u, v, prm);
  acc.newton += r.iters;
  if (r.status != ROOT_ACCEPTED) return;
  for (int k = 0; k < acc.n; ++k)
    if (fabs(acc.t[k] - r.t) < prm.dedup) return;
  if (acc.n >= kMaxRoots) {
    acc.flags |= FLAG_RESHOOT;
    return;
  }
  const int k = acc.n++;
  acc.t[k] = r.t;
  acc.chi += r.sign;
  if (r.tang || r.graze) acc.flags |= FLAG_RESHOOT;
  if (r.onsurf) acc.flags |= FLAG_ONSURF;
  if constexpr (kRecord) {
    acc.u[k] = r.u;
    acc.v[k] = r.v;
    acc.sign[k] = r.sign;
    acc.tang[k] = r.tang;
    acc.graze[k] = r.graze;
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
  int32_t chi = r.chi, fl = r.flags;
  const bool tail = seg_reduce(slot, chi, fl);
  if (slot >= 0 && tail) {
    if (chi) atomicAdd(&chi_acc[slot], chi);
    if (fl) atomicOr(&flag_acc[slot], fl);
  }
  warp_add_u64(&counters[CNT_NODES], (unsigned long long)r.nodes);
  warp_add_u64(&counters[CNT_NEWTON], (unsigned long long)r.newton);
  warp_add_u64(&counters[CNT_ROOTS], (unsigned long long)r.roots);
}

cudaError_t launch_intersect_dfs(const gwn_scene* sc, const Round& rd, int64_t npairs,
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
