// gwn_k3.cuh -- K3 work items and the per-candidate leaf test, shared by
// the fused cull (gwn_cull.cu, K2 + K3 pass 0) and the K3 passes
// (gwn_wavefront.cu).
#pragma once

#include "gwn_dfs.cuh"

namespace gwn {

struct NodeItem {
  int32_t slot;   // query slot of the round
  int32_t leaf;   // round leaf index (patch, fold tree)
  uint64_t code;  // level:6 | iu:29 | iv:29
};

// Self-contained Newton work item (one coalesced 64-byte load): the query
// slot, the patch, the leaf code for ownership, the certified start and the
// query's ray-frame projection.
struct alignas(16) NewtonItem {
  int32_t slot;
  int32_t patch;
  uint64_t code;
  double u, v;
  double qa, qb, qc;
  double pad;
};


// warp-aggregated append: returns the slot or -1 if over capacity
__device__ __forceinline__ long long warp_push(bool want, unsigned long long* counter,
                                               unsigned long long cap, int* overflow) {
  unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!want) return -1;
  unsigned long long idx = base + __popc(mask & ((1u << lane) - 1));
  if (idx >= cap) {
    *overflow = 1;
    return -1;
  }
  return (long long)idx;
}

// Block-aggregated reservation in two append queues: one atomic per queue
// per call instead of one per warp.  Every warp of a kernel hammering the same
// counter serialises at its L2 slice: the SHFL waiting for that atomic was
// 30% of k3_candidates' and 15% of the cull's stall samples at config 2.
// n0 / n1: this thread's item counts; o0 / o1: its first slots.  Every thread
// of the block must call it (three barriers; the shared block is reusable on
// return).  A null counter reserves nothing.
template <int NW>
struct BlockPush {
  unsigned long long cnt[2][NW];
  unsigned long long base[2];
};

template <int NW>
__device__ __forceinline__ void block_reserve(BlockPush<NW>& S, int n0, int n1,
                                              unsigned long long* c0, unsigned long long* c1,
                                              unsigned long long& o0, unsigned long long& o1) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int i0 = n0, i1 = n1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v0 = __shfl_up_sync(0xffffffffu, i0, o);
    const int v1 = __shfl_up_sync(0xffffffffu, i1, o);
    if (lane >= o) {
      i0 += v0;
      i1 += v1;
    }
  }
  if (lane == 31) {
    S.cnt[0][wid] = (unsigned long long)i0;
    S.cnt[1][wid] = (unsigned long long)i1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {  // thread q reserves queue q
    const int q = threadIdx.x;
    unsigned long long run = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const unsigned long long t = S.cnt[q][k];
      S.cnt[q][k] = run;
      run += t;
    }
    unsigned long long* c = q ? c1 : c0;
    S.base[q] = (run && c) ? atomicAdd(c, run) : 0ull;
  }
  __syncthreads();
  o0 = S.base[0] + S.cnt[0][wid] + (unsigned long long)(i0 - n0);
  o1 = S.base[1] + S.cnt[1][wid] + (unsigned long long)(i1 - n1);
  __syncthreads();
}

__device__ __forceinline__ void warp_sum_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Candidate test of query (qa, qb) against a leaf / sub-leaf record:
// 0 exclude, 1 certified root (Newton start nu, nv), 2 undecided.
__device__ __forceinline__ int leaf_test(const LeafRec& L, double qa, double qb,
                                         const DevParams& prm, double& nu, double& nv) {
  const double span = 1.0 + 2.0 * kLeafM;
  const double tl = kLeafM / span, th = (1.0 + kLeafM) / span;
  const int lev = code_level(L.code);
  const double wu = code_wu(lev), wv = code_wv(lev);
  const double u0 = (double)code_iu(L.code) * wu, v0 = (double)code_iv(L.code) * wv;
  const double tol = prm.domain_tol;
  const double xlo_u = tl - (u0 == 0.0 ? tol / (wu * span) : 0.0);
  const double xhi_u = th + (u0 + wu == 1.0 ? tol / (wu * span) : 0.0);
  const double xlo_v = tl - (v0 == 0.0 ? tol / (wv * span) : 0.0);
  const double xhi_v = th + (v0 + wv == 1.0 ? tol / (wv * span) : 0.0);
  KrawPre k;
  k.Ga = L.Ga; k.Gb = L.Gb;
  k.Y00 = L.Y00; k.Y01 = L.Y01; k.Y10 = L.Y10; k.Y11 = L.Y11;
  k.R0 = L.R0; k.R1 = L.R1;
  k.ok = L.ok != 0;
  double s0, s1;
  int kr = kraw_query(k, L.Ga - qa, L.Gb - qb, xlo_u, xhi_u, xlo_v, xhi_v, -1e-7, 1.0 + 1e-7,
                      s0, s1);
  if (kr == 2) {  // separating axes of the leaf hull (rigorous exclusion)
    const double p1 = L.n1a * qa + L.n1b * qb, p2 = L.n2a * qa + L.n2b * qb;
    if (p1 < L.lo1 || p1 > L.hi1 || p2 < L.lo2 || p2 > L.hi2) kr = 0;
  }
  if (kr == 1) {
    nu = u0 - kLeafM * wu + s0 * span * wu;
    nv = v0 - kLeafM * wv + s1 * span * wv;
  }
  return kr;
}

// leaf_test reading the record through a pointer, in two steps: the
// Krawczyk data (64 B) and code/patch/ok (16 B) first, the separating axes
// (64 B) only for the undecided candidates -- most are settled by the first
// step, which halves the record traffic of K3 pass 0.
__device__ __forceinline__ int leaf_test_lazy(const LeafRec* __restrict__ Lp, double qa,
                                              double qb, const DevParams& prm, double& nu,
                                              double& nv, int32_t& patch, uint64_t& code) {
  const double2* p = reinterpret_cast<const double2*>(Lp);
  const double2 g = __ldg(p), y0 = __ldg(p + 1), y1 = __ldg(p + 2), r = __ldg(p + 3);
  const double2 tail = __ldg(p + 8);
  code = (uint64_t)__double_as_longlong(tail.x);
  const long long po = __double_as_longlong(tail.y);
  patch = (int32_t)(po & 0xffffffffll);
  const int32_t ok = (int32_t)(po >> 32);
  const double span = 1.0 + 2.0 * kLeafM;
  const double tl = kLeafM / span, th = (1.0 + kLeafM) / span;
  const int lev = code_level(code);
  const double wu = code_wu(lev), wv = code_wv(lev);
  const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
  const double tol = prm.domain_tol;
  const double xlo_u = tl - (u0 == 0.0 ? tol / (wu * span) : 0.0);
  const double xhi_u = th + (u0 + wu == 1.0 ? tol / (wu * span) : 0.0);
  const double xlo_v = tl - (v0 == 0.0 ? tol / (wv * span) : 0.0);
  const double xhi_v = th + (v0 + wv == 1.0 ? tol / (wv * span) : 0.0);
  KrawPre k;
  k.Ga = g.x; k.Gb = g.y;
  k.Y00 = y0.x; k.Y01 = y0.y; k.Y10 = y1.x; k.Y11 = y1.y;
  k.R0 = r.x; k.R1 = r.y;
  k.ok = ok != 0;
  double s0, s1;
  int kr = kraw_query(k, g.x - qa, g.y - qb, xlo_u, xhi_u, xlo_v, xhi_v, -1e-7, 1.0 + 1e-7,
                      s0, s1);
  if (kr == 2) {  // separating axes of the leaf hull (rigorous exclusion)
    const double2 a0 = __ldg(p + 4), a1 = __ldg(p + 5), a2 = __ldg(p + 6), a3 = __ldg(p + 7);
    const double p1 = a0.x * qa + a0.y * qb, p2 = a2.x * qa + a2.y * qb;
    if (p1 < a1.x || p1 > a1.y || p2 < a3.x || p2 > a3.y) kr = 0;
  }
  if (kr == 1) {
    nu = u0 - kLeafM * wu + s0 * span * wu;
    nv = v0 - kLeafM * wv + s1 * span * wv;
  }
  return kr;
}

// K3 queues: the cull's (query, leaf) candidates; after the candidate test
// the undecided ones for the subdivision fallback, certified ones for the
// Newton pass.  Each candidate yields at most one item, so every queue has
// cap = the candidate capacity of the round.
struct K3Queues {
  int2* pairs;  // (query slot, leaf) candidates from the cull
  NodeItem* fq;
  unsigned long long* f_count;
  NewtonItem* nq;
  unsigned long long* n_count;
  unsigned long long cap;
  int* overflow;
  // Patch bins (scenes beyond the shared-memory patch table, n_bins = P, else
  // 0): k3_candidates counts its Newton items per patch (bin_count, zeroed per
  // round) and records (patch, rank in bin) per item; k_bin_scan /
  // k_bin_scatter turn that into `perm`, the item indices in patch order, so a
  // warp of the Newton pass works on one patch at a time.
  int2* nkey = nullptr;
  int32_t* perm = nullptr;
  int32_t* bin_count = nullptr;
  int32_t* bin_off = nullptr;
  int32_t n_bins = 0;
};

}  // namespace gwn
