// gwn_dfs.cuh -- per-thread depth-first root enumeration below one node of a
// patch's subdivision tree (the single-ray all_hits API and the rare K3
// fallback items whose leaf test was undecided).
//
// Every node is tested exactly like a K1 leaf: Krawczyk over the node box
// expanded by kLeafM on each side (query-independent part from the expanded
// net, then the query step), so a root anywhere in the node -- including on
// a split line -- certifies as soon as the node is small enough; roots count
// only in the node whose half-open box owns them.  Nodes that still do not
// certify kDfsDepth levels below the start node contain a near-tangent
// double root (a silhouette fold of the projection): the query is flagged
// for a new direction, the reference's policy for tangent rays
// (surfaces.py:696).
#pragma once

#include "gwn_patch.cuh"

namespace gwn {

// A line meets a bicubic patch in at most 2*3*3 = 18 points (Bezout), so the
// record path never truncates a root set.
constexpr int kMaxRoots = 18;
constexpr int kDfsDepth = 12;   // levels below the start node before re-shooting
constexpr int kDfsBudget = 512; // nodes per item before re-shooting

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
// surfaces.py:668 tolerance band): dedup across neighbouring nodes.
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
  o.lo_u = own_lo(u0, tol);
  o.hi_u = own_hi(u1, tol);
  o.lo_v = own_lo(v0, tol);
  o.hi_v = own_hi(v1, tol);
  o.closed_u = u1 == 1.0;
  o.closed_v = v1 == 1.0;
  return o;
}

// Per-pair constants of the node test.
struct NodeCtx {
  const double* P48;
  double qa, qb, qc;
  double eps_box;
};

__device__ __forceinline__ NodeCtx node_ctx(const double* __restrict__ P48, double qa, double qb,
                                            double qc, const DevParams& prm) {
  double amag = 0.0, alo = INFINITY, ahi = -INFINITY, blo = INFINITY, bhi = -INFINITY;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double A = __ldg(P48 + k), B = __ldg(P48 + 16 + k);
    amag = fmax(amag, fmax(fabs(A), fabs(B)));
    alo = fmin(alo, A); ahi = fmax(ahi, A); blo = fmin(blo, B); bhi = fmax(bhi, B);
  }
  NodeCtx c;
  c.P48 = P48;
  c.qa = qa;
  c.qb = qb;
  c.qc = qc;
  c.eps_box = 1e-12 * (1.0 + amag) + 3.0 * prm.domain_tol * fmax(ahi - alo, bhi - blo);
  return c;
}

enum : int { NODE_EXCLUDED = 0, NODE_ROOT = 1, NODE_SPLIT = 2, NODE_AMBIGUOUS = 3 };

// One node of the subdivision tree: control-box and separating-axis tests of
// the node's own piece, then Krawczyk over the node box expanded by kLeafM.
// NODE_ROOT: r holds the Newton result and `owned` says whether this node's
// half-open box owns it (r.status tells acceptance); a Newton that left the
// certified box comes back as NODE_AMBIGUOUS.
__device__ __forceinline__ int node_test(const NodeCtx& c, uint64_t code, int max_level,
                                         const DevParams& prm, RootResult& r, bool& owned) {
  const double tol = prm.domain_tol;
  const double span = 1.0 + 2.0 * kLeafM;
  const double tl = kLeafM / span, th = (1.0 + kLeafM) / span;
  const int L = code_level(code);
  const double wu = code_wu(L), wv = code_wv(L);
  const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
  double a[16], b[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    a[k] = __ldg(c.P48 + k);
    b[k] = __ldg(c.P48 + 16 + k);
  }
  extract_net(a, u0, u0 + wu, v0, v0 + wv);
  extract_net(b, u0, u0 + wu, v0, v0 + wv);
  double la = a[0], ha = a[0], lb = b[0], hb = b[0];
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    la = fmin(la, a[k]); ha = fmax(ha, a[k]);
    lb = fmin(lb, b[k]); hb = fmax(hb, b[k]);
  }
  const double e = c.eps_box;
  if (la - e > c.qa || ha + e < c.qa || lb - e > c.qb || hb + e < c.qb) return NODE_EXCLUDED;
  // separating axes normal to the node's centre tangents: near a silhouette
  // fold the node's image is a thin strip the axis-aligned box bounds poorly
  if (!hull_sat(a, b, c.qa, c.qb, e)) return NODE_EXCLUDED;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    a[k] = __ldg(c.P48 + k);
    b[k] = __ldg(c.P48 + 16 + k);
  }
  const double eu0 = u0 - kLeafM * wu, eu1 = u0 + (1.0 + kLeafM) * wu;
  const double ev0 = v0 - kLeafM * wv, ev1 = v0 + (1.0 + kLeafM) * wv;
  extract_net(a, eu0, eu1, ev0, ev1);
  extract_net(b, eu0, eu1, ev0, ev1);
  const KrawPre kp = kraw_pre(a, b);
  const double xlo_u = tl - (u0 == 0.0 ? tol / (wu * span) : 0.0);
  const double xhi_u = th + (u0 + wu == 1.0 ? tol / (wu * span) : 0.0);
  const double xlo_v = tl - (v0 == 0.0 ? tol / (wv * span) : 0.0);
  const double xhi_v = th + (v0 + wv == 1.0 ? tol / (wv * span) : 0.0);
  double s0, s1;
  const int kr = kraw_query(kp, kp.Ga - c.qa, kp.Gb - c.qb, xlo_u, xhi_u, xlo_v, xhi_v, -1e-7,
                            1.0 + 1e-7, s0, s1);
  if (kr == 0) return NODE_EXCLUDED;
  if (kr == 1) {
    r = newton_solve(c.P48, c.qa, c.qb, c.qc, eu0 + s0 * span * wu, ev0 + s1 * span * wv, prm);
    if (r.status == ROOT_DIVERGED) return NODE_AMBIGUOUS;
    const double mu = 1e-6 * wu, mv = 1e-6 * wv;
    if (r.u < eu0 - mu || r.u > eu1 + mu || r.v < ev0 - mv || r.v > ev1 + mv)
      return NODE_AMBIGUOUS;  // Newton left the certified basin
    owned = own_box_of(code, tol).has(r.u, r.v);
    return NODE_ROOT;
  }
  if (L >= max_level) return NODE_AMBIGUOUS;  // near-tangent double root
  return NODE_SPLIT;
}

__device__ __forceinline__ void child_codes(uint64_t code, uint64_t& c0, uint64_t& c1) {
  const int L = code_level(code);
  const uint64_t iu = code_iu(code), iv = code_iv(code);
  if ((L & 1) == 0) {
    c0 = make_code(L + 1, 2 * iu, iv);
    c1 = make_code(L + 1, 2 * iu + 1, iv);
  } else {
    c0 = make_code(L + 1, iu, 2 * iv);
    c1 = make_code(L + 1, iu, 2 * iv + 1);
  }
}

// Append an accepted root unless it duplicates one already found
// (surfaces.py:672-674: ray points closer than eps.dedup).
template <bool kRecord>
__device__ __forceinline__ void record_root(RootAcc<kRecord>& acc, const RootResult& r,
                                            const DevParams& prm) {
  for (int k = 0; k < acc.n; ++k)
    if (fabs(acc.t[k] - r.t) < prm.dedup) return;
  if (acc.n >= kMaxRoots) {  // more than Bezout's bound: only from a budget overrun
    acc.flags |= FLAG_RESHOOT | FLAG_OVERFLOW;
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

// All roots of one (query, patch) pair below the start node `start`
// (0 = the whole patch), depth-first on one thread (single-ray all_hits).
template <bool kRecord>
__device__ PairOut solve_pair(const double* __restrict__ P48, double qa, double qb, double qc,
                              const DevParams& prm, uint64_t start, int depth,
                              RootAcc<kRecord>& acc) {
  const NodeCtx ctx = node_ctx(P48, qa, qb, qc, prm);
  const int max_level = min(code_level(start) + depth, kMaxLevel);
  const int budget = depth >= kMaxLevel ? kNodeBudget : kDfsBudget;
  acc.n = 0;
  acc.chi = 0;
  acc.flags = 0;
  acc.newton = 0;
  int nodes = 0;
  uint64_t stack[2 * kMaxLevel + 4];
  int top = 0;
  stack[top++] = start;
  while (top > 0) {
    const uint64_t code = stack[--top];
    if (++nodes > budget) {
      acc.flags |= FLAG_RESHOOT;
      break;
    }
    RootResult r;
    bool owned = false;
    const int o = node_test(ctx, code, max_level, prm, r, owned);
    if (o == NODE_AMBIGUOUS) {
      acc.flags |= FLAG_RESHOOT;
      if constexpr (kRecord) {
        // An undecided node below the depth cap holds a near-tangent double
        // root (silhouette fold).  The reference reports such a contact as a
        // record with tangency set (surfaces.py:684-687,696), which makes the
        // caller re-shoot: solve from the node centre and record the contact
        // as tangent (node centre and t = C - p.d if Newton does not settle).
        const int L = code_level(code);
        const double wu = code_wu(L), wv = code_wv(L);
        const double uc = ((double)code_iu(code) + 0.5) * wu;
        const double vc = ((double)code_iv(code) + 0.5) * wv;
        RootResult q = newton_solve(P48, qa, qb, qc, uc, vc, prm);
        acc.newton += q.iters;
        if (q.status != ROOT_ACCEPTED) {
          double bu[4], dbu[4], bv[4], dbv[4], C, Cu, Cv;
          bern3(uc, bu, dbu);
          bern3(vc, bv, dbv);
          eval_coord(P48 + 32, bu, dbu, bv, dbv, C, Cu, Cv);
          q.u = uc;
          q.v = vc;
          q.t = C - qc;
          q.sign = 1;
          q.graze = 1;
          if (q.t < -prm.t_tol) continue;
        }
        q.tang = 1;
        record_root(acc, q, prm);
      }
    } else if (o == NODE_ROOT) {
      acc.newton += r.iters;
      if (r.status != ROOT_ACCEPTED || !owned) continue;
      record_root(acc, r, prm);
    } else if (o == NODE_SPLIT) {
      uint64_t c0, c1;
      child_codes(code, c0, c1);
      stack[top++] = c1;
      stack[top++] = c0;
    }
  }
  PairOut out;
  out.chi = acc.chi;
  out.flags = acc.flags;
  out.nodes = nodes;
  out.newton = acc.newton;
  out.roots = acc.n;
  return out;
}

}  // namespace gwn
