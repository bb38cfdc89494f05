// gwn_cull.cu -- K2: query x leaf cull in the ray frame of the round.
//
// Replaces the reference's per-(ray, patch) `patch.aabb()` + ray_aabb_clip
// (surfaces.py:636-639, geometry.py:198-219): with every ray of the round
// parallel to d, a leaf sub-patch can be hit only if the query's projection
// (p.e1, p.e2) lies in the leaf's projected control box and the leaf reaches
// past p along d (cmax >= p.d).  Point location is a uniform grid of packed
// float boxes (rounded outward, so the float test keeps every true
// candidate), or the LBVH when the grid would not stay compact.
//
// One pass: each thread collects its leaves in a small register buffer, then
// the warp reserves space for all lanes with a single atomic (warp prefix
// sum), so the (slot, leaf) candidates of a query are contiguous; queries
// with more than kLBuf candidates append the rest one by one.  The kernel
// counts every candidate; if the round's capacity was too small the engine
// re-runs the round with the exact size.  (Fusing the candidate test into
// this kernel was measured slower: its registers cut the occupancy the
// latency-bound cell walk needs.)
#include <stdlib.h>

#include "gwn_k3.cuh"

namespace gwn {

constexpr int kStack = 64;  // >= LBVH depth bound (30-bit Morton + 32-bit index tie-break)
// Per-thread candidate buffer (local memory, L1-resident).  A query with more
// candidates appends the rest one atomic at a time, each a full L2 round trip
// the lane waits for: with 12 entries that spill path was 74% of the grid
// cull's stall samples at config 5 (rays through many overlapping surfaces
// have 20-60 candidates).  Measured at config 5, 2^23 queries: 12 entries
// 5.99 ms, 24 4.21, 32 3.33, 48 2.26, 64 1.92, 96 1.83, 128 1.90; config 4
// 2.03 -> 1.22 ms; config 2 unchanged.
#ifndef GWN_CULL_LBUF
#define GWN_CULL_LBUF 64
#endif
constexpr int kLBuf = GWN_CULL_LBUF;

__device__ __forceinline__ void query_proj(const Frame& f, const double* __restrict__ pos,
                                           int32_t q, double& qa, double& qb, double& qc) {
  double x = pos[3 * (int64_t)q], y = pos[3 * (int64_t)q + 1], z = pos[3 * (int64_t)q + 2];
  qa = x * f.e1[0] + y * f.e1[1] + z * f.e1[2];
  qb = x * f.e2[0] + y * f.e2[1] + z * f.e2[2];
  qc = x * f.d[0] + y * f.d[1] + z * f.d[2];
}

struct GridView {
  const int32_t* offs;
  const CellEnt* ent;
  int32_t na, nb;
  double x0, y0, ia, ib;
};

// Grid path with warp-level load balancing: when a warp's cell lists are
// long or skewed, the lanes' ranges are prefix-summed across the warp and
// the warp walks the concatenated (query, entry) list 32 tests at a time,
// each lane finding its query by a shuffle binary search -- every lane busy
// instead of waiting for the longest list.  Short even lists keep the
// per-lane walk (cheaper without the shuffles).  Measured (threshold 32 of
// 8/16/24/32/64): config 5 cull 174 -> 82 us, config 3 159 -> 117 us,
// config 4 3.3 -> 2.95 ms, config 2 unchanged.
#ifndef GWN_CULL_BS
#define GWN_CULL_BS 128
#endif
#ifndef GWN_CULL_MINB
#define GWN_CULL_MINB 1
#endif
__global__ void __launch_bounds__(GWN_CULL_BS, GWN_CULL_MINB)
k_cull_grid(GridView grid, Frame f, int32_t m, const int32_t* __restrict__ active,
            const double* __restrict__ pos, double* __restrict__ qproj,
            int2* __restrict__ pairs, unsigned long long* __restrict__ pair_count,
            unsigned long long cap, CullZero z) {
  // programmatic dependent launch: K3's candidate test (which waits for this
  // grid's completion before reading) may launch once the last wave of cull
  // blocks is running, filling SMs as they retire
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int beg = 0, cnt = 0;
  float fqa = 0.f, fqb = 0.f, fqc = 0.f;
  if (s < m) {
    if (z.chi) z.chi[s] = 0;
    if (z.flags) z.flags[s] = 0;
    const int32_t q = active ? active[s] : s;
    double qa, qb, qc;
    query_proj(f, pos, q, qa, qb, qc);
    qproj[3 * (int64_t)s] = qa;
    qproj[3 * (int64_t)s + 1] = qb;
    qproj[3 * (int64_t)s + 2] = qc;
    const double fa = (qa - grid.x0) * grid.ia, fb = (qb - grid.y0) * grid.ib;
    if (fa >= 0.0 && fb >= 0.0 && fa < (double)grid.na && fb < (double)grid.nb) {
      const int c = (int)fb * grid.na + (int)fa;
      beg = __ldg(grid.offs + c);
      cnt = __ldg(grid.offs + c + 1) - beg;
    }
    // fp32 compares on the rounded query are a superset of the fp64 test:
    // qa >= lo implies fl(qa) >= fl(lo) >= lo rounded down
    fqa = (float)qa;
    fqb = (float)qb;
    fqc = (float)qc;
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  // short lists (<= GWN_CULL_MX) or even ones (per-lane walk at >= 50% lane
  // efficiency): each lane walks its own cell; long and skewed lists: the
  // balanced walk below
  const int mx = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
#ifndef GWN_CULL_MX
#define GWN_CULL_MX 32
#endif
  if (mx <= GWN_CULL_MX || 32 * mx <= 2 * total + 64) {
    const int32_t me = blockIdx.x * blockDim.x + threadIdx.x;
    int buf[kLBuf];
    int n = 0;
    auto take = [&](float2 e0, float2 e1, float2 e2) {
      if (fqa >= e0.x && fqa <= e0.y && fqb >= e1.x && fqb <= e1.y && e2.x >= fqc) {
        const int leaf = __float_as_int(e2.y);
        if (n < kLBuf) {
          buf[n++] = leaf;
        } else {  // spill: rare, append individually
          const unsigned long long k = atomicAdd(pair_count, 1ull);
          if (k < cap) pairs[k] = make_int2(me, leaf);
        }
      }
    };
    // entries in groups of GWN_CULL_BATCH: every load of a group is issued
    // before its first test, so one L1/L2 round trip covers the group
#ifndef GWN_CULL_BATCH
#define GWN_CULL_BATCH 4
#endif
    int j = 0;
    for (; j + GWN_CULL_BATCH <= cnt; j += GWN_CULL_BATCH) {
      float2 E[GWN_CULL_BATCH][3];
#pragma unroll
      for (int u = 0; u < GWN_CULL_BATCH; ++u) {
        const float2* p = reinterpret_cast<const float2*>(grid.ent + beg + j + u);
        E[u][0] = __ldg(p);
        E[u][1] = __ldg(p + 1);
        E[u][2] = __ldg(p + 2);
      }
#pragma unroll
      for (int u = 0; u < GWN_CULL_BATCH; ++u) take(E[u][0], E[u][1], E[u][2]);
    }
    for (; j < cnt; ++j) {
      const float2* p = reinterpret_cast<const float2*>(grid.ent + beg + j);
      take(__ldg(p), __ldg(p + 1), __ldg(p + 2));
    }
    // one warp-aggregated reservation for the buffered candidates
    int hincl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, hincl, o);
      if (lane >= o) hincl += v;
    }
    const int htot = __shfl_sync(0xffffffffu, hincl, 31);
    unsigned long long base = 0;
    if (lane == 31 && htot) base = atomicAdd(pair_count, (unsigned long long)htot);
    base = __shfl_sync(0xffffffffu, base, 31);
    const unsigned long long o0 = base + (unsigned long long)(hincl - n);
    for (int k = 0; k < n; ++k)
      if (o0 + k < cap) pairs[o0 + k] = make_int2(me, buf[k]);
    return;
  }
  for (int k0 = 0; k0 < total; k0 += 32) {
    const int k = k0 + lane;
    bool hit = false;
    int leaf = 0;
    // first lane whose inclusive prefix exceeds k (every lane shuffles; lanes
    // past the end search for the last entry and stay idle)
    const int kk = k < total ? k : total - 1;
    int src = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int v = __shfl_sync(0xffffffffu, incl, src + step - 1);
      if (v <= kk) src += step;
    }
    // gather the owner's query and range (all lanes take part in shuffles)
    const float ga = __shfl_sync(0xffffffffu, fqa, src), gb = __shfl_sync(0xffffffffu, fqb, src),
                gc = __shfl_sync(0xffffffffu, fqc, src);
    const int gbeg = __shfl_sync(0xffffffffu, beg, src);
    const int gexcl = __shfl_sync(0xffffffffu, incl - cnt, src);
    if (k < total) {
      const int e = gbeg + (k - gexcl);
      const float2* p = reinterpret_cast<const float2*>(grid.ent + e);
      const float2 e0 = __ldg(p), e1 = __ldg(p + 1), e2 = __ldg(p + 2);
      hit = ga >= e0.x && ga <= e0.y && gb >= e1.x && gb <= e1.y && e2.x >= gc;
      leaf = __float_as_int(e2.y);
    }
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(pair_count, (unsigned long long)__popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (hit) {
        const unsigned long long o = base + __popc(mask & ((1u << lane) - 1));
        if (o < cap) pairs[o] = make_int2(blockIdx.x * blockDim.x + (threadIdx.x & ~31) + src, leaf);
      }
    }
  }
}

__global__ void __launch_bounds__(128)
k_cull(const Node* __restrict__ nodes, const double* __restrict__ leafbox, int64_t n_leaves,
       GridView grid, Frame f, int32_t m, const int32_t* __restrict__ active,
       const double* __restrict__ pos, double* __restrict__ qproj,
       int2* __restrict__ pairs, unsigned long long* __restrict__ pair_count,
       unsigned long long cap, CullZero z) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = s < m;
  int buf[kLBuf];
  int n = 0;
  double qa = 0.0, qb = 0.0, qc = 0.0;
  if (live) {
    // the round's per-slot accumulators start at zero (K3/K4 run after K2)
    if (z.chi) z.chi[s] = 0;
    if (z.flags) z.flags[s] = 0;
    const int32_t q = active ? active[s] : s;
    query_proj(f, pos, q, qa, qb, qc);
    qproj[3 * (int64_t)s] = qa;
    qproj[3 * (int64_t)s + 1] = qb;
    qproj[3 * (int64_t)s + 2] = qc;
    auto emit = [&](int leaf) {
      if (n < kLBuf) {
        buf[n++] = leaf;
      } else {  // spill: rare, append individually
        const unsigned long long k = atomicAdd(pair_count, 1ull);
        if (k < cap) pairs[k] = make_int2(s, leaf);
      }
    };
    if (grid.offs) {
      // uniform grid: one cell, a short list of packed float boxes
      const double fa = (qa - grid.x0) * grid.ia, fb = (qb - grid.y0) * grid.ib;
      if (fa >= 0.0 && fb >= 0.0 && fa < (double)grid.na && fb < (double)grid.nb) {
        const int c = (int)fb * grid.na + (int)fa;
        const int k1 = __ldg(grid.offs + c + 1);
        // float compares on the rounded query are a superset of the double
        // test: qa >= lo implies fl(qa) >= fl(lo) >= lo rounded down
        const float fqa = (float)qa, fqb = (float)qb, fqc = (float)qc;
        for (int k = __ldg(grid.offs + c); k < k1; ++k) {
          const float2* e = reinterpret_cast<const float2*>(grid.ent + k);
          const float2 e0 = __ldg(e), e1 = __ldg(e + 1), e2 = __ldg(e + 2);
          if (fqa >= e0.x && fqa <= e0.y && fqb >= e1.x && fqb <= e1.y && e2.x >= fqc)
            emit(__float_as_int(e2.y));
        }
      }
    } else if (n_leaves == 1) {
      const double* b = leafbox;
      if (qa >= b[0] && qa <= b[1] && qb >= b[2] && qb <= b[3] && b[4] >= qc) emit(0);
    } else {
      int stack[kStack];
      int top = 0;
      int node = 0;
      bool dropped = false;
      for (;;) {
        const Node& nd = nodes[node];
        int next = -1;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const bool hit = qa >= nd.alo[c] && qa <= nd.ahi[c] && qb >= nd.blo[c] &&
                           qb <= nd.bhi[c] && nd.cmax[c] >= qc;
          if (!hit) continue;
          const int ch = nd.child[c];
          if (ch < 0) emit(~ch);
          else if (next < 0) next = ch;
          else if (top < kStack) stack[top++] = ch;
          else dropped = true;  // unreachable (kStack >= the LBVH depth bound); never silent
        }
        if (next >= 0) node = next;
        else if (top > 0) node = stack[--top];
        else break;
      }
      // a subtree that could not be stacked: the query takes a new direction
      // (this thread zeroed flags[s] above; K3 / K4 only OR into it later)
      if (dropped && z.flags) z.flags[s] = FLAG_RESHOOT;
    }
  }
  // warp-aggregated reservation of the buffered candidates
  const int lane = threadIdx.x & 31;
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && total) base = atomicAdd(pair_count, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 31);
  const unsigned long long o0 = base + (unsigned long long)(incl - n);
  for (int k = 0; k < n; ++k)
    if (o0 + k < cap) pairs[o0 + k] = make_int2(s, buf[k]);
}

cudaError_t launch_cull(const gwn_scene* sc, const Round& rd, int32_t m, const int32_t* active,
                        const double* pos, double* qproj, unsigned long long* pair_count,
                        int64_t cap, CullZero z, const K3Queues& Q, unsigned long long* counters,
                        cudaStream_t st) {
  (void)sc;
  (void)counters;
  if (m <= 0) return cudaSuccess;
  GridView g{rd.use_grid ? rd.cell_offs : nullptr, rd.cell_ent, rd.ga, rd.gb,
             rd.gx0, rd.gy0, rd.gia, rd.gib};
  if (g.offs) {
    k_cull_grid<<<(m + GWN_CULL_BS - 1) / GWN_CULL_BS, GWN_CULL_BS, 0, st>>>(g, rd.f, m, active, pos, qproj, Q.pairs,
                                                 pair_count, (unsigned long long)cap, z);
    return cudaGetLastError();
  }
  k_cull<<<(m + 127) / 128, 128, 0, st>>>(rd.nodes, rd.leafbox, rd.n_leaves, g, rd.f, m, active,
                                          pos, qproj, Q.pairs, pair_count,
                                          (unsigned long long)cap, z);
  return cudaGetLastError();
}

}  // namespace gwn
