// gwn_wavefront.cu -- K3 as a level-synchronous wavefront over subdivision
// nodes (the batched intersector; the per-pair DFS of gwn_intersect.cu stays
// for the single-ray all_hits API).
//
// Why: a per-pair depth-first search leaves ~80% of the lanes of a warp idle
// (ncu, round 1: 6.6 active threads / warp) because pairs need 1..40 nodes.
// Here one work item is one node (pair, level, iu, iv):
//   * the node's 2-D net is rebuilt from the pair's root net by the same
//     de Casteljau halvings the DFS applies (bit-identical nets),
//   * the Krawczyk test classifies it: exclude / certified unique root /
//     split; split children pass a control-box test before they are queued
//     (warp-aggregated compaction of the surviving candidates),
//   * certified nodes become Newton items, solved in a separate uniform pass.
// Dedup of a root found from two neighbouring certified nodes (their
// certification boxes overlap by 1e-7) is by ownership: a root counts only in
// the node whose half-open parameter box contains it (the domain edge nodes
// own the surfaces.py:668 tolerance band).  Per-query chi / flags are then
// reduced with a segmented warp-shuffle reduction keyed by query slot.
#include "gwn_patch.cuh"

namespace gwn {

struct NodeItem {
  int32_t pair;
  int32_t pad;
  uint64_t code;  // level:6 | iu:29 | iv:29
};

struct NewtonItem {
  int32_t pair;
  int32_t kind;   // 0: certified node, 1: level cap, 2: certified leaf (expanded box)
  uint64_t code;
  double u, v;
};


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

// origin-in-control-box test of both children of a split along dir,
// streamed without materialising the children
__device__ __forceinline__ void child_boxes(const double* a, const double* b, int dir, double eps,
                                            bool& okL, bool& okR) {
  double aLmin = INFINITY, aLmax = -INFINITY, aRmin = INFINITY, aRmax = -INFINITY;
  double bLmin = INFINITY, bLmax = -INFINITY, bRmin = INFINITY, bRmax = -INFINITY;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int i0 = dir == 0 ? l : 4 * l;
    const int st = dir == 0 ? 4 : 1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double* x = c == 0 ? a : b;
      double p0 = x[i0], p1 = x[i0 + st], p2 = x[i0 + 2 * st], p3 = x[i0 + 3 * st];
      double a01 = 0.5 * (p0 + p1), a12 = 0.5 * (p1 + p2), a23 = 0.5 * (p2 + p3);
      double b0 = 0.5 * (a01 + a12), b1 = 0.5 * (a12 + a23);
      double m = 0.5 * (b0 + b1);
      double lmin = fmin(fmin(p0, a01), fmin(b0, m)), lmax = fmax(fmax(p0, a01), fmax(b0, m));
      double rmin = fmin(fmin(m, b1), fmin(a23, p3)), rmax = fmax(fmax(m, b1), fmax(a23, p3));
      if (c == 0) {
        aLmin = fmin(aLmin, lmin); aLmax = fmax(aLmax, lmax);
        aRmin = fmin(aRmin, rmin); aRmax = fmax(aRmax, rmax);
      } else {
        bLmin = fmin(bLmin, lmin); bLmax = fmax(bLmax, lmax);
        bRmin = fmin(bRmin, rmin); bRmax = fmax(bRmax, rmax);
      }
    }
  }
  okL = aLmin <= eps && aLmax >= -eps && bLmin <= eps && bLmax >= -eps;
  okR = aRmin <= eps && aRmax >= -eps && bRmin <= eps && bRmax >= -eps;
}

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

__device__ __forceinline__ void warp_sum_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

struct WaveArgs {
  const int32_t* pair_slot;
  int32_t* pair_patch;
  const double* qproj;
  const double* proj;
  DevParams prm;
  int32_t* chi;
  int32_t* flags;
  int32_t* pair_nodes;
  unsigned long long* counters;
  int* overflow;
  NewtonItem* nq;
  unsigned long long* n_count;
  unsigned long long n_cap;
};

// K3 pass 0: one thread per (query, leaf) candidate.  The leaf's Krawczyk
// data are query-independent (K1), so the test is ~20 flops: exclude,
// certified (-> Newton item) or undecided (-> node wavefront from the leaf).
__global__ void __launch_bounds__(128)
k3_candidates(int64_t npairs, const int32_t* __restrict__ pair_leaf,
              const LeafRec* __restrict__ leaves, NodeItem* __restrict__ out,
              unsigned long long* __restrict__ out_count, unsigned long long out_cap, WaveArgs w) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long tested = 0;
  // leaf box D inside the expanded certification box D' (local coords t)
  const double span = 1.0 + 2.0 * kLeafM;
  const double tl = kLeafM / span, th = (1.0 + kLeafM) / span;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < npairs; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool wantN = false, wantF = false;
    int32_t pair = (int32_t)i;
    uint64_t code = 0;
    double nu_ = 0.0, nv_ = 0.0;
    if (i < npairs) {
      const LeafRec L = leaves[pair_leaf[i]];
      w.pair_patch[i] = L.patch;
      code = L.code;
      const int32_t slot = w.pair_slot[i];
      const double qa = w.qproj[3 * (int64_t)slot], qb = w.qproj[3 * (int64_t)slot + 1];
      ++tested;
      const int lev = code_level(code);
      const double wu = code_wu(lev), wv = code_wv(lev);
      const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
      const double tol = w.prm.domain_tol;
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
      const int kr = kraw_query(k, L.Ga - qa, L.Gb - qb, xlo_u, xhi_u, xlo_v, xhi_v, -1e-7,
                                1.0 + 1e-7, s0, s1);
      if (kr == 1) {
        wantN = true;
        nu_ = u0 - kLeafM * wu + s0 * span * wu;
        nv_ = v0 - kLeafM * wv + s1 * span * wv;
      } else if (kr == 2) {
        wantF = true;
      }
    }
    long long k = warp_push(wantF, out_count, out_cap, w.overflow);
    if (k >= 0) out[k] = NodeItem{pair, 0, code};
    k = warp_push(wantN, w.n_count, w.n_cap, w.overflow);
    if (k >= 0) w.nq[k] = NewtonItem{pair, 2, code, nu_, nv_};
  }
  warp_sum_u64(&w.counters[CNT_NODES], tested);
}

// One wavefront pass over undecided nodes (each item carries its own level).
__global__ void __launch_bounds__(128)
k3_level(const NodeItem* __restrict__ in, const unsigned long long* __restrict__ in_count,
         NodeItem* __restrict__ out, unsigned long long* __restrict__ out_count,
         unsigned long long out_cap, WaveArgs w) {
  const int64_t n = (int64_t)*in_count;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long nodes = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool live = i < n;
    int32_t pair = 0;
    uint64_t code = 0;
    if (live) {
      NodeItem it = in[i];
      pair = it.pair;
      code = it.code;
    }
    const int level = code_level(code);
    const uint64_t iu = code_iu(code), iv = code_iv(code);
    bool wantL = false, wantR = false, wantN = false;
    int kind = 0;
    double nu_ = 0.0, nv_ = 0.0;
    if (live) {
      const int32_t slot = w.pair_slot[pair];
      const double* P48 = w.proj + 48 * (int64_t)w.pair_patch[pair];
      const double qa = w.qproj[3 * (int64_t)slot], qb = w.qproj[3 * (int64_t)slot + 1];
      RootNet rn;
      load_root(P48, qa, qb, w.prm, rn);
      ++nodes;
      rebuild(rn.a, rn.b, level, iu, iv);
      const double wu = code_wu(level), wv = code_wv(level);
      const double u0 = (double)iu * wu, v0 = (double)iv * wv;
      const double tol = w.prm.domain_tol;
      const double xlo_u = u0 == 0.0 ? -tol / wu : 0.0;
      const double xhi_u = u0 + wu == 1.0 ? 1.0 + tol / wu : 1.0;
      const double xlo_v = v0 == 0.0 ? -tol / wv : 0.0;
      const double xhi_v = v0 + wv == 1.0 ? 1.0 + tol / wv : 1.0;
      double s0, s1;
      const int kr = krawczyk(rn.a, rn.b, xlo_u, xhi_u, xlo_v, xhi_v, s0, s1);
      if (kr == 1) {
        wantN = true;
        nu_ = u0 + s0 * wu;
        nv_ = v0 + s1 * wv;
      } else if (kr == 2) {
        if (level >= kMaxLevel) {
          wantN = true;
          kind = 1;
          nu_ = u0 + 0.5 * wu;
          nv_ = v0 + 0.5 * wv;
        } else {
          child_boxes(rn.a, rn.b, level & 1, rn.eps_box, wantL, wantR);
          const int add = (int)wantL + (int)wantR;
          if (add && atomicAdd(&w.pair_nodes[pair], add) + add > kNodeBudget) {
            atomicOr(&w.flags[slot], FLAG_RESHOOT);  // tangent-like explosion: re-shoot
            wantL = wantR = false;
          }
        }
      }
    }
    // warp-aggregated compaction of survivors (all lanes converge here)
    const int dir = level & 1;
    const uint64_t ciuL = dir == 0 ? 2 * iu : iu, civL = dir == 0 ? iv : 2 * iv;
    const uint64_t ciuR = dir == 0 ? 2 * iu + 1 : iu, civR = dir == 0 ? iv : 2 * iv + 1;
    long long k = warp_push(wantL, out_count, out_cap, w.overflow);
    if (k >= 0) out[k] = NodeItem{pair, 0, make_code(level + 1, ciuL, civL)};
    k = warp_push(wantR, out_count, out_cap, w.overflow);
    if (k >= 0) out[k] = NodeItem{pair, 0, make_code(level + 1, ciuR, civR)};
    k = warp_push(wantN, w.n_count, w.n_cap, w.overflow);
    if (k >= 0) w.nq[k] = NewtonItem{pair, kind, code, nu_, nv_};
  }
  warp_sum_u64(&w.counters[CNT_NODES], nodes);
}

// Newton pass over the certified / level-cap nodes + ownership + K5 part 1.
__global__ void __launch_bounds__(128) k3_newton(WaveArgs w) {
  const int64_t n = (int64_t)*w.n_count;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long iters = 0, roots = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    int32_t slot = -1, chi = 0, fl = 0;
    if (i < n) {
      const NewtonItem it = w.nq[i];
      slot = w.pair_slot[it.pair];
      const double* P48 = w.proj + 48 * (int64_t)w.pair_patch[it.pair];
      const double* q = w.qproj + 3 * (int64_t)slot;
      RootResult r = newton_solve(P48, q[0], q[1], q[2], it.u, it.v, w.prm);
      iters += r.iters;
      const int level = code_level(it.code);
      const double wu = ldexp(1.0, -((level + 1) >> 1));
      const double wv = ldexp(1.0, -(level >> 1));
      const double u0 = (double)code_iu(it.code) * wu, v0 = (double)code_iv(it.code) * wv;
      const double u1 = u0 + wu, v1 = v0 + wv;
      const double tol = w.prm.domain_tol;
      if (r.status == ROOT_DIVERGED) {
        if (it.kind != 1) fl |= FLAG_RESHOOT;  // certified root not reached: re-shoot
      } else {
        // half-open ownership box (domain edges own the tolerance band)
        const double lo_u = u0 == 0.0 ? -tol : u0, hi_u = u1 == 1.0 ? 1.0 + tol : u1;
        const double lo_v = v0 == 0.0 ? -tol : v0, hi_v = v1 == 1.0 ? 1.0 + tol : v1;
        const bool own = r.u >= lo_u && (r.u < hi_u || (u1 == 1.0 && r.u <= hi_u)) &&
                         r.v >= lo_v && (r.v < hi_v || (v1 == 1.0 && r.v <= hi_v));
        if (own) {
          if (r.status == ROOT_ACCEPTED) {
            ++roots;
            chi = r.sign;
            if (r.tang || r.graze) fl |= FLAG_RESHOOT;
            if (r.onsurf) fl |= FLAG_ONSURF;
          }
        } else if (it.kind != 1) {
          // certified: the unique root lies in the certification box (node
          // +1e-7, or the kLeafM-expanded leaf box); farther away means Newton
          // left the certified basin
          const double ex = it.kind == 2 ? kLeafM + 1e-6 : 2e-7;
          const double mu = ex * wu, mv = ex * wv;
          if (r.u < u0 - mu || r.u > u1 + mu || r.v < v0 - mv || r.v > v1 + mv)
            fl |= FLAG_RESHOOT;
        } else {
          // level cap: a root well outside this tiny node belongs elsewhere
          if (r.status == ROOT_ACCEPTED && fabs(r.u - 0.5 * (u0 + u1)) < 2.0 * wu &&
              fabs(r.v - 0.5 * (v0 + v1)) < 2.0 * wv) {
            // a neighbour owns it
          }
        }
      }
    }
    // segmented warp-shuffle reduction keyed by query slot, one atomic per run
    const bool tail = seg_reduce(slot, chi, fl);
    if (slot >= 0 && tail) {
      if (chi) atomicAdd(&w.chi[slot], chi);
      if (fl) atomicOr(&w.flags[slot], fl);
    }
  }
  warp_sum_u64(&w.counters[CNT_NEWTON], iters);
  warp_sum_u64(&w.counters[CNT_ROOTS], roots);
}

static int grid_for(const void* fn, int sm_count) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 128, 0);
  if (per_sm < 1) per_sm = 1;
  return sm_count * per_sm;
}

// K3 driver: levels run in batches of 4 between host checks of the frontier
// size; queue overflow (never seen in practice) clears the accumulators of
// the m active queries and retries with doubled capacity.
cudaError_t launch_intersect(const gwn_scene* sc, const Round& rd, int64_t npairs,
                             const int32_t* pair_slot, const int32_t* pair_leaf,
                             const double* qproj, int32_t* chi, int32_t* flags, int32_t m,
                             unsigned long long* counters, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  static thread_local int g_cand = 0, g_level = 0, g_newton = 0, g_dev = -1;
  static thread_local unsigned long long* h = nullptr;
  if (g_dev != sc->device) {
    g_cand = grid_for((const void*)k3_candidates, sc->sm_count);
    g_level = grid_for((const void*)k3_level, sc->sm_count);
    g_newton = grid_for((const void*)k3_newton, sc->sm_count);
    g_dev = sc->device;
  }
  cudaError_t e = cudaSuccess;
  if (!h && (e = cudaMallocHost(&h, sizeof(unsigned long long) * 4)) != cudaSuccess) return e;
  unsigned long long cap = (unsigned long long)(npairs + 4096);
  unsigned long long ncap = (unsigned long long)(npairs + 4096);
  for (int attempt = 0; attempt < 8; ++attempt) {
    NodeItem *qa = nullptr, *qb = nullptr;
    NewtonItem* nq = nullptr;
    unsigned long long* cnt = nullptr;  // [0],[1] node queues, [2] newton, [3] overflow
    int32_t *pn = nullptr, *pp = nullptr;
    bool overflow = false;
#define WC(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)
    WC(cudaMallocAsync(&qa, sizeof(NodeItem) * cap, st));
    WC(cudaMallocAsync(&qb, sizeof(NodeItem) * cap, st));
    WC(cudaMallocAsync(&nq, sizeof(NewtonItem) * ncap, st));
    WC(cudaMallocAsync(&cnt, sizeof(unsigned long long) * 4, st));
    WC(cudaMallocAsync(&pn, sizeof(int32_t) * npairs, st));
    WC(cudaMallocAsync(&pp, sizeof(int32_t) * npairs, st));
    WC(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 4, st));
    WC(cudaMemsetAsync(pn, 0, sizeof(int32_t) * npairs, st));
    {
      WaveArgs w{pair_slot, pp, qproj, rd.proj, sc->dprm, chi, flags, pn,
                 counters, (int*)(cnt + 3), nq, cnt + 2, ncap};
      NodeItem* bufs[2] = {qa, qb};
      k3_candidates<<<g_cand, 128, 0, st>>>(npairs, pair_leaf, rd.leaves, qa, cnt, cap, w);
      WC(cudaGetLastError());
      WC(cudaMemcpyAsync(h, cnt, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, st));
      WC(cudaStreamSynchronize(st));
      bool more = h[0] > 0 && !h[3];
      int pass = 0;
      while (more && pass <= kMaxLevel) {
        for (int k = 0; k < 4 && pass <= kMaxLevel; ++k, ++pass) {
          unsigned long long* out_c = cnt + ((pass + 1) & 1);
          WC(cudaMemsetAsync(out_c, 0, sizeof(unsigned long long), st));
          k3_level<<<g_level, 128, 0, st>>>(bufs[pass & 1], cnt + (pass & 1),
                                            bufs[(pass + 1) & 1], out_c, cap, w);
          WC(cudaGetLastError());
        }
        WC(cudaMemcpyAsync(h, cnt, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, st));
        WC(cudaStreamSynchronize(st));
        more = h[pass & 1] > 0 && !h[3];
      }
      overflow = h[3] != 0;
      if (!overflow) {
        k3_newton<<<g_newton, 128, 0, st>>>(w);
        WC(cudaGetLastError());
      }
    }
  out:
    if (qa) cudaFreeAsync(qa, st);
    if (qb) cudaFreeAsync(qb, st);
    if (nq) cudaFreeAsync(nq, st);
    if (cnt) cudaFreeAsync(cnt, st);
    if (pn) cudaFreeAsync(pn, st);
    if (pp) cudaFreeAsync(pp, st);
#undef WC
    if (e != cudaSuccess) return e;
    if (!overflow) return cudaSuccess;
    if ((e = cudaMemsetAsync(chi, 0, sizeof(int32_t) * m, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(flags, 0, sizeof(int32_t) * m, st)) != cudaSuccess) return e;
    cap *= 2;
    ncap *= 2;
  }
  return cudaErrorMemoryAllocation;
}

}  // namespace gwn
