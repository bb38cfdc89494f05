// gwn_dfs.cuh -- per-thread depth-first root enumeration below one node
// (the single-ray all_hits API and the rare K3 fallback items).
#pragma once

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

// Parameter box that owns roots (half-open; the domain edges own the
// surfaces.py:668 tolerance band): dedup across neighbouring start nodes.
struct OwnBox {
  double lo_u, hi_u, lo_v, hi_v;
  bool closed_u, closed_v;
  __device__ __forceinline__ bool has(double u, double v) const {
    return u >= lo_u && (u < hi_u || (closed_u && u <= hi_u)) && v >= lo_v &&
           (v < hi_v || (closed_v && v <= hi_v));
  }
};

__device__ __forceinline__ OwnBox own_box_of(uint64_t code, double tol) {
  const int L = code_level(code);
  const double wu = code_wu(L), wv = code_wv(L);
  const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
  const double u1 = u0 + wu, v1 = v0 + wv;
  OwnBox o;
  o.lo_u = u0 == 0.0 ? -tol : u0;
  o.hi_u = u1 == 1.0 ? 1.0 + tol : u1;
  o.lo_v = v0 == 0.0 ? -tol : v0;
  o.hi_v = v1 == 1.0 ? 1.0 + tol : v1;
  o.closed_u = u1 == 1.0;
  o.closed_v = v1 == 1.0;
  return o;
}

// Newton on the whole patch from (u,v); on acceptance record the root with
// the reference's 1e-9 dedup (surfaces.py:672-674), if the start node's
// ownership box holds it.
template <bool kRecord>
__device__ void newton_root(const double* __restrict__ P48, double qa, double qb, double qc,
                            double u, double v, const DevParams& prm, const OwnBox& own,
                            RootAcc<kRecord>& acc) {
  RootResult r = newton_solve(P48, qa, qb, qc, u, v, prm);
  acc.newton += r.iters;
  if (r.status != ROOT_ACCEPTED) return;
  if (!own.has(r.u, r.v)) return;
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

// Complete depth-first root enumeration for one (query, patch) pair below the
// start node `start` (0 = the whole patch); roots count only inside the start
// node's ownership box.
template <bool kRecord>
__device__ PairOut solve_pair(const double* __restrict__ P48, double qa, double qb, double qc,
                              const DevParams& prm, uint64_t start, RootAcc<kRecord>& acc) {
  RootNet rn;
  load_root(P48, qa, qb, prm, rn);
  double* a = rn.a;
  double* b = rn.b;
  const double eps_box = rn.eps_box;
  const OwnBox own = own_box_of(start, prm.domain_tol);
  int level = code_level(start);
  rebuild(a, b, level, code_iu(start), code_iv(start));
  acc.n = 0;
  acc.chi = 0;
  acc.flags = 0;
  acc.newton = 0;
  int nodes = 0;
  double st_a[kStackNets][16], st_b[kStackNets][16];
  double st_box[kStackNets][3];  // u0, v0, level
  int top = 0;
  double u0 = (double)code_iu(start) * code_wu(level), v0 = (double)code_iv(start) * code_wv(level);
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
      newton_root(P48, qa, qb, qc, u0 + s0 * wu, v0 + s1 * wv, prm, own, acc);
    } else if (kr == 2) {
      if (level >= kMaxLevel) {
        newton_root(P48, qa, qb, qc, u0 + 0.5 * wu, v0 + 0.5 * wv, prm, own, acc);
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

}  // namespace gwn
