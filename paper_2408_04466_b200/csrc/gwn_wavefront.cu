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
#include "gwn_k3.cuh"

namespace gwn {

struct WaveArgs {
  const LeafRec* leaves;  // round leaves (patch of a fallback item)
  const double* qproj;
  const double* proj;
  const double* powc;   // proj in the power basis (Newton pass)
  DevParams prm;
  int32_t* chi;
  int32_t* flags;
  HitRec* rec;          // record mode (ray reuse): every owned root, else nullptr
  unsigned long long* rec_count;
  unsigned long long rec_cap;
  unsigned long long* counters;
  int* overflow;
  NewtonItem* nq;
  unsigned long long* n_count;
  unsigned long long n_cap;
  unsigned long long* n_work;  // Newton work counter (dynamic fetch), zeroed per round
  // fold trees of the round (Round::sub*), sub_offs null when there are none
  const int64_t* sub_offs;
  const LeafRec* sub;
  const double* subbox;
  const int32_t* subskip;
  const int4* subgc;
  int32_t sub_level;
};

// Newton solve of a certified (leaf or fold sub-leaf) candidate + ownership:
// adds the owned root's sign to chi and its flags to fl.
__device__ __forceinline__ void newton_own(const WaveArgs& w, int32_t slot, uint64_t code,
                                           const RootResult& r, int32_t& chi, int32_t& fl,
                                           unsigned long long& iters,
                                           unsigned long long& roots) {
  iters += r.iters;
  const int level = code_level(code);
  const double wu = code_wu(level), wv = code_wv(level);
  const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
  const double u1 = u0 + wu, v1 = v0 + wv;
  const double tol = w.prm.domain_tol;
  // the unique root lies in the certification box (leaf box expanded by
  // kLeafM); landing farther away means Newton left the certified basin
  const double ex = kLeafM + 1e-6;
  const bool in_cert = r.u >= u0 - ex * wu && r.u <= u1 + ex * wu && r.v >= v0 - ex * wv &&
                       r.v <= v1 + ex * wv;
  if (r.status == ROOT_DIVERGED || !in_cert) {
    fl |= FLAG_RESHOOT;  // certified root not reached: re-shoot
  } else if (r.status == ROOT_ACCEPTED) {
    // half-open ownership box (domain edges own the tolerance band)
    const double lo_u = own_lo(u0, tol), hi_u = own_hi(u1, tol);
    const double lo_v = own_lo(v0, tol), hi_v = own_hi(v1, tol);
    const bool own = r.u >= lo_u && (r.u < hi_u || (u1 == 1.0 && r.u <= hi_u)) &&
                     r.v >= lo_v && (r.v < hi_v || (v1 == 1.0 && r.v <= hi_v));
    if (own) {
      ++roots;
      chi += r.sign;
      if (r.tang || r.graze) fl |= FLAG_RESHOOT;
      if (r.onsurf) fl |= FLAG_ONSURF;
      if (w.rec) {
        const unsigned long long k = atomicAdd(w.rec_count, 1ull);
        if (k < w.rec_cap) w.rec[k] = HitRec{slot, r.sign, r.t};
        else fl |= FLAG_RESHOOT;
      }
    }
  }
}

__device__ __forceinline__ void newton_accept(const WaveArgs& w, int32_t slot, int32_t patch,
                                              uint64_t code, double u, double v, double qa,
                                              double qb, double qc, int32_t& chi, int32_t& fl,
                                              unsigned long long& iters,
                                              unsigned long long& roots) {
  const double* P48 = w.proj + 48 * (int64_t)patch;
  const RootResult r = newton_solve(P48, qa, qb, qc, u, v, w.prm);
  newton_own(w, slot, code, r, chi, fl, iters, roots);
}

// K3 pass 0: one thread per (query, leaf) candidate.  The leaf's Krawczyk
// data are query-independent (K1), so the test is ~40 flops: exclude,
// certified (-> Newton item) or undecided (-> fallback item).
constexpr int kCandBlock = 256;

#ifndef GWN_CAND_MINB
#define GWN_CAND_MINB 3
#endif
__global__ void __launch_bounds__(kCandBlock, GWN_CAND_MINB)
k3_candidates(const unsigned long long* __restrict__ npairs_dev, K3Queues Q, WaveArgs w) {
  __shared__ BlockPush<kCandBlock / 32> S;
  // launched programmatically behind the cull (GWN_PDL): wait for its results
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // on capacity overflow the engine discards and re-runs the round; never
  // read past the buffers
  const int64_t npairs = (int64_t)min(*npairs_dev, Q.cap);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long tested = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < npairs; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool wantN = false, wantF = false;
    int32_t slot = 0, patch = 0, leaf = 0;
    uint64_t code = 0;
    double nu_ = 0.0, nv_ = 0.0, qa = 0.0, qb = 0.0, qc = 0.0;
    if (i < npairs) {
      const int2 pr = Q.pairs[i];
      slot = pr.x;
      leaf = pr.y;
      qa = w.qproj[3 * (int64_t)slot];
      qb = w.qproj[3 * (int64_t)slot + 1];
      qc = w.qproj[3 * (int64_t)slot + 2];
      ++tested;
      const int kr = leaf_test_lazy(w.leaves + leaf, qa, qb, w.prm, nu_, nv_, patch, code);
      wantN = kr == 1;
      wantF = kr == 2;
    }
    // Patch bins: rank of the item in its patch's bin, one atomic per distinct
    // patch of the warp (neighbouring rays cross the same patches), issued
    // before the block reservation so its round trip overlaps the barriers.
    // (Every tested pair yields at most one item and at most `cap` pairs are
    // tested, so a Newton item always has a slot: kn < cap below.)
    unsigned grp = 0;
    int32_t rank0 = 0;
    const int lane = threadIdx.x & 31;
    if (Q.n_bins) {
      grp = __match_any_sync(0xffffffffu, wantN ? patch : -1 - lane);
      if (wantN && lane == __ffs(grp) - 1) rank0 = atomicAdd(Q.bin_count + patch, __popc(grp));
    }
    // (the loop bound is block-uniform, so every thread reaches the barriers)
    unsigned long long kf = 0, kn = 0;
    block_reserve(S, wantF ? 1 : 0, wantN ? 1 : 0, Q.f_count, Q.n_count, kf, kn);
    if (wantF) {
      if (kf < Q.cap) Q.fq[kf] = NodeItem{slot, leaf, code};
      else *Q.overflow = 1;
    }
    if (wantN) {
      if (kn < Q.cap) Q.nq[kn] = NewtonItem{slot, patch, code, nu_, nv_, qa, qb, qc, 0.0};
      else *Q.overflow = 1;
    }
    if (Q.n_bins && wantN) {
      rank0 = __shfl_sync(grp, rank0, __ffs(grp) - 1);
      if (kn < Q.cap)
        Q.nkey[kn] = make_int2(patch, rank0 + __popc(grp & ((1u << lane) - 1u)));
    }
  }
  warp_sum_u64(&w.counters[CNT_NODES], tested);
}

// Undecided leaves (rays near a silhouette fold of the projection):
// breadth-first below the leaf with a frontier shared by a batch of items per
// warp; the lanes test frontier entries of any item in parallel.  Items per
// warp = ceil(items / warps), at most 32: few items stay spread over the
// GPU, many items keep every lane busy.  A frontier entry is either
//   * a node of the leaf's precomputed fold tree (K1, k_foldtree): box and
//     separating-axis test from stored data, certified sub-leaves solved by
//     Newton in place, the fold's own sub-leaves handed on as codes; or
//   * a subdivision code: node_test (gwn_dfs.cuh) derives the node's net.
// Roots count only in the node that owns them; undecidable nodes below the
// depth cap flag the query for a new direction.
constexpr int kFrontier = 512;
constexpr int kFbWarps = 4;  // warps per block
constexpr uint8_t kTreeTag = 0x80;  // fi tag: entry is a fold-tree node index

__global__ void __launch_bounds__(32 * kFbWarps)
k3_fallback(const NodeItem* __restrict__ in, const unsigned long long* __restrict__ in_count,
            WaveArgs w) {
  __shared__ uint64_t fr[kFbWarps][2][kFrontier];
  __shared__ uint8_t fi[kFbWarps][2][kFrontier];
  __shared__ double iq[kFbWarps][32][4];  // qa, qb, qc, eps_box
  __shared__ int32_t islot[kFbWarps][32], ipatch[kFbWarps][32], imax[kFbWarps][32];
  __shared__ int32_t ichi[kFbWarps][32], ifl[kFbWarps][32], inodes[kFbWarps][32];
  __shared__ int32_t s_n0[kFbWarps];  // initial frontier size
  // programmatic dependent launch (GWN_PDL): the Newton pass queued behind this
  // kernel on the same stream may start as soon as every fallback block is
  // resident -- it does not read the fallback's results
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t n = (int64_t)min(*in_count, w.n_cap);  // pushes past capacity were dropped
  const int lane = threadIdx.x & 31, wb = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const long long want = (long long)((n + nwarps - 1) / nwarps);
  const int ipw = (int)(want < 1 ? 1 : want > 32 ? 32 : want);
  unsigned long long nodes = 0, iters = 0, roots = 0;
  for (int64_t b0 = warp * ipw; b0 < n; b0 += nwarps * ipw) {
    const int nb = (int)min((int64_t)ipw, n - b0);
    if (lane == 0) s_n0[wb] = 0;
    __syncwarp();
    if (lane < nb) {
      const NodeItem it = in[b0 + lane];
      const int32_t slot = it.slot;
      const int32_t patch = w.leaves[it.leaf].patch;
      const double* q = w.qproj + 3 * (int64_t)slot;
      const NodeCtx c = node_ctx(w.proj + 48 * (int64_t)patch, q[0], q[1], q[2], w.prm);
      iq[wb][lane][0] = c.qa;
      iq[wb][lane][1] = c.qb;
      iq[wb][lane][2] = c.qc;
      iq[wb][lane][3] = c.eps_box;
      islot[wb][lane] = slot;
      ipatch[wb][lane] = patch;
      imax[wb][lane] = min(max(code_level(it.code) + kDfsDepth, w.sub_level + 4), kMaxLevel);
      ichi[wb][lane] = 0;
      ifl[wb][lane] = 0;
      inodes[wb][lane] = 0;
      const int64_t t0 = w.sub_offs ? w.sub_offs[it.leaf] : 0;
      const int64_t t1 = w.sub_offs ? w.sub_offs[it.leaf + 1] : 0;
      if (t1 > t0) {  // the two subtrees of the leaf's fold tree
        const int64_t t0b = t0 + w.subskip[t0];
        const int pos = atomicAdd(&s_n0[wb], t0b < t1 ? 2 : 1);  // <= 64 <= kFrontier
        fr[wb][0][pos] = (uint64_t)t0;
        fi[wb][0][pos] = (uint8_t)(lane | kTreeTag);
        if (t0b < t1) {
          fr[wb][0][pos + 1] = (uint64_t)t0b;
          fi[wb][0][pos + 1] = (uint8_t)(lane | kTreeTag);
        }
      } else {
        const int pos = atomicAdd(&s_n0[wb], 1);
        fr[wb][0][pos] = it.code;
        fi[wb][0][pos] = (uint8_t)lane;
      }
    }
    __syncwarp();
    int cur = 0, ncur = s_n0[wb], levels = 0;
    const long long tclk0 = clock64();
    int tree_lv = 0, code_lv = 0;
    while (ncur > 0) {
      ++levels;
      {
        bool hc = false, ht = false;
        for (int k = lane; k < ncur; k += 32) {
          if (fi[wb][cur][k] & kTreeTag) ht = true; else hc = true;
        }
        if (__any_sync(0xffffffffu, hc)) ++code_lv;
        if (__any_sync(0xffffffffu, ht)) ++tree_lv;
      }
      int nnext = 0;
      for (int base = 0; base < ncur; base += 32) {
        const int k = base + lane;
        int nout = 0, item = 0;
        uint8_t otag = 0;
        uint64_t out0 = 0, out1 = 0, out2 = 0, out3 = 0;
        if (k < ncur) {
          const uint64_t e = fr[wb][cur][k];
          const uint8_t tg = fi[wb][cur][k];
          item = tg & 0x7f;
          const double qa = iq[wb][item][0], qb = iq[wb][item][1], qc = iq[wb][item][2];
          ++nodes;
          if (tg & kTreeTag) {
            // precomputed fold-tree node
            const int64_t t = (int64_t)e;
            // every load of the node up front (one memory round trip per
            // level): box, skips of the node and of its first child, record
            const double* bx = w.subbox + 5 * t;
            const int32_t sk = __ldg(w.subskip + t);
            const int4 gc = w.subgc[t];
            const double b0 = __ldg(bx), b1 = __ldg(bx + 1), b2 = __ldg(bx + 2),
                         b3 = __ldg(bx + 3), b4 = __ldg(bx + 4);
            const LeafRec S = w.sub[t];
            if (qa >= b0 && qa <= b1 && qb >= b2 && qb <= b3 && b4 >= qc) {
              if (sk == 1) {
                double su = 0.0, sv = 0.0;
                const int kr = leaf_test(S, qa, qb, w.prm, su, sv);
                if (kr == 1) {
                  int32_t cchi = 0, cfl = 0;
                  newton_accept(w, islot[wb][item], ipatch[wb][item], S.code, su, sv, qa, qb, qc,
                                cchi, cfl, iters, roots);
                  if (cchi) atomicAdd(&ichi[wb][item], cchi);
                  if (cfl) atomicOr(&ifl[wb][item], cfl);
                } else if (kr == 2) {  // on the fold itself: subdivide from here
                  nout = 1;
                  out0 = S.code;
                }
              } else {
                const double p1 = S.n1a * qa + S.n1b * qb, p2 = S.n2a * qa + S.n2b * qb;
                if (!(p1 < S.lo1 || p1 > S.hi1 || p2 < S.lo2 || p2 > S.hi2)) {
                  // grandchildren (a leaf child stands for itself)
                  otag = kTreeTag;
                  nout = 2 + (gc.z >= 0) + (gc.w >= 0);
                  out0 = (uint64_t)(t + gc.x);
                  out1 = (uint64_t)(t + gc.y);
                  out2 = (uint64_t)(t + gc.z);
                  out3 = (uint64_t)(t + gc.w);
                }
              }
            }
          } else {
            NodeCtx c;
            c.P48 = w.proj + 48 * (int64_t)ipatch[wb][item];
            c.qa = qa;
            c.qb = qb;
            c.qc = qc;
            c.eps_box = iq[wb][item][3];
            RootResult r;
            bool owned = false;
            int o = node_test(c, e, imax[wb][item], w.prm, r, owned);
            if (atomicAdd(&inodes[wb][item], 1) >= kDfsBudget) {
              o = NODE_AMBIGUOUS;  // budget: give up on this direction
            }
            if (o == NODE_AMBIGUOUS) {
              atomicOr(&ifl[wb][item], FLAG_RESHOOT);
            } else if (o == NODE_ROOT) {
              iters += r.iters;
              if (r.status == ROOT_ACCEPTED && owned) {
                ++roots;
                atomicAdd(&ichi[wb][item], r.sign);
                int f = 0;
                if (r.tang || r.graze) f |= FLAG_RESHOOT;
                if (r.onsurf) f |= FLAG_ONSURF;
                if (w.rec) {
                  const unsigned long long kk = atomicAdd(w.rec_count, 1ull);
                  if (kk < w.rec_cap) w.rec[kk] = HitRec{islot[wb][item], r.sign, r.t};
                  else f |= FLAG_RESHOOT;
                }
                if (f) atomicOr(&ifl[wb][item], f);
              }
            } else if (o == NODE_SPLIT) {
              nout = 2;
              child_codes(e, out0, out1);
            }
          }
        }
        // warp-aggregated append of 0..4 entries per lane (inclusive scan)
        int incl = nout;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (nout) {
          const int pos = nnext + incl - nout;
          if (pos + nout <= kFrontier) {
            const uint64_t outs[4] = {out0, out1, out2, out3};
            for (int q = 0; q < nout; ++q) {
              fr[wb][cur ^ 1][pos + q] = outs[q];
              fi[wb][cur ^ 1][pos + q] = (uint8_t)(item | otag);
            }
          } else {
            atomicOr(&ifl[wb][item], FLAG_RESHOOT);  // frontier overflow
          }
        }
        nnext = min(nnext + tot, kFrontier);
      }
      __syncwarp();
      cur ^= 1;
      ncur = nnext;
    }
    __syncwarp();
    if (lane < nb) {
      const int32_t slot = islot[wb][lane];
      if (ichi[wb][lane]) atomicAdd(&w.chi[slot], ichi[wb][lane]);
      if (ifl[wb][lane]) atomicOr(&w.flags[slot], ifl[wb][lane]);
      // diagnostics: largest item, items beyond 16 nodes
      const int nn = inodes[wb][lane];
      atomicMax(&w.counters[CNT_MAXNODES], (unsigned long long)nn);
      (void)nn;
      if (lane == 0) atomicMax(&w.counters[CNT_MAXLEVELS], (unsigned long long)levels);
      if (lane == 0) {
        const long long dt = clock64() - tclk0;
        // debug: slowest warp batch: cycles | tree levels | code levels | items
        const unsigned long long key = ((unsigned long long)(dt > 0 ? dt : 0) << 24) |
                                       ((unsigned long long)tree_lv << 16) |
                                       ((unsigned long long)code_lv << 8) | (unsigned long long)nb;
        atomicMax(&w.counters[CNT_BIGITEMS], key);
      }
    }
    __syncwarp();
  }
  warp_sum_u64(&w.counters[CNT_NODES], nodes);
  warp_sum_u64(&w.counters[CNT_NEWTON], iters);
  warp_sum_u64(&w.counters[CNT_ROOTS], roots);
}

// Newton pass over the certified leaves + ownership + K5 part 1.
//
// Dynamic fetch, 32 items per warp: blocks that start late (the fallback
// kernel holds part of every SM) find the queue drained instead of owning a
// fixed share of it.  The fetch is software-pipelined one batch deep: the
// atomic that reserves batch b+1 and the loads of its items are issued before
// batch b is solved, so neither the atomic's round trip nor the item load sits
// on the critical path.  (Measured at config 2: the stall samples move to the
// coefficient loads; the step time is unchanged, the pipeline is kept.)
// Scenes of at most kTabMaxP patches read the coefficients from a shared
// memory table (k3_newton<true>): no registers hold them, so more warps fit.
#ifndef GWN_NEWTON_MINB
#define GWN_NEWTON_MINB 3
#endif
#ifndef GWN_NEWTON_MINB_SMEM
#define GWN_NEWTON_MINB_SMEM 5
#endif
#ifndef GWN_NEWTON_BERNSTEIN
#define GWN_NEWTON_BERNSTEIN 0
#endif
// Patch table in shared memory (P <= kTabMaxP): power coefficients at a
// padded stride, so lanes reading the same coefficient of different patches
// hit different banks (100 words per patch: bank offset 4 per patch).
constexpr int kTabStride = 50;
constexpr int kTabMaxP = 96;  // 38.4 KB

template <bool kSmem>
__device__ __forceinline__ void newton_item_run(const WaveArgs& w, const double* tab,
                                                const NewtonItem& it, int32_t& chi, int32_t& fl,
                                                unsigned long long& iters,
                                                unsigned long long& roots) {
#if GWN_NEWTON_BERNSTEIN
  const double* P48 = w.proj + 48 * (int64_t)it.patch;
  RootResult r = newton_solve(P48, it.qa, it.qb, it.qc, it.u, it.v, w.prm);
#else
  const double* W48 = kSmem ? tab + kTabStride * it.patch : w.powc + 48 * (int64_t)it.patch;
  RootResult r = newton_solve_pow<kSmem ? 2 : 0>(W48, it.qa, it.qb, it.qc, it.u, it.v, w.prm);
#endif
  newton_own(w, it.slot, it.code, r, chi, fl, iters, roots);
}

// Work-counter reservation.  nvcc/ptxas expand atomicAdd (inline-PTX
// atom.add too) into a warp-aggregated sequence whose SHFL consumes the
// result at once, which put the atomic's round trip back on the critical
// path (13.5% of the stall samples at config 2 with the pipelined fetch).
// atom.inc with a limit the counter never reaches is left alone (ptxas turns
// a 0xffffffff limit back into an add), so the counter counts 32-item batches
// (low word of n_work, zeroed per round) and the result is consumed a batch
// later.
// Returns the batch index; the caller scales it by 32 only where it is
// consumed (a multiply right after the atomic waits for its round trip:
// 36% of the stall samples when reserve_batch returned 32 * old).
__device__ __forceinline__ unsigned reserve_batch(unsigned long long* p) {
  unsigned old;
  asm volatile("atom.global.inc.u32 %0, [%1], %2;"
               : "=r"(old) : "l"(p), "r"(0x7fffffffu) : "memory");
  return old;
}

template <bool kSmem>
__global__ void __launch_bounds__(128, kSmem ? GWN_NEWTON_MINB_SMEM : GWN_NEWTON_MINB)
k3_newton(WaveArgs w, int32_t P) {
  extern __shared__ double tab[];
  if (kSmem) {
    for (int k = threadIdx.x; k < 48 * P; k += blockDim.x)
      tab[kTabStride * (k / 48) + k % 48] = w.powc[k];
    __syncthreads();
  }
  const int64_t n = (int64_t)min(*w.n_count, w.n_cap);
  unsigned long long iters = 0, roots = 0;
  const int lane = threadIdx.x & 31;
  unsigned b_cur = 0, b_nxt = 0;  // batch indices (32 items each)
  if (lane == 0) {
    b_cur = reserve_batch(w.n_work);
    b_nxt = reserve_batch(w.n_work);
  }
  int64_t base = 32 * (int64_t)__shfl_sync(0xffffffffu, b_cur, 0);
  NewtonItem it{};
  if (base + lane < n) it = w.nq[base + lane];
  while (base < n) {
    // reservations are monotone, so the next batch starts past this one and
    // every reserved batch below n is solved
    const int64_t nbase = 32 * (int64_t)__shfl_sync(0xffffffffu, b_nxt, 0);
    NewtonItem nx{};
    if (nbase + lane < n) nx = w.nq[nbase + lane];
    if (lane == 0 && nbase < n) b_nxt = reserve_batch(w.n_work);
    int32_t slot = -1, chi = 0, fl = 0;
    if (base + lane < n) {
      slot = it.slot;
      newton_item_run<kSmem>(w, tab, it, chi, fl, iters, roots);
    }
    // segmented warp-shuffle reduction keyed by query slot, one atomic per run
    const bool tail = seg_reduce(slot, chi, fl);
    if (slot >= 0 && tail) {
      if (chi) atomicAdd(&w.chi[slot], chi);
      if (fl) atomicOr(&w.flags[slot], fl);
    }
    it = nx;
    base = nbase;
  }
  // Programmatic dependent of k3_fallback (which triggers on entry): wait for
  // the fallback grid here, after the work loop, so Newton keeps its overlap
  // with it and Newton's completion implies the fallback's (its chi / flag
  // atomics are then ordered before K4, K5 and the next round by stream
  // order).  A no-op when launched without the attribute.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  warp_sum_u64(&w.counters[CNT_NEWTON], iters);
  warp_sum_u64(&w.counters[CNT_ROOTS], roots);
}

// Patch bins, step 2: exclusive scan of the per-patch item counts (one block;
// P is at most a few 10^4).
__global__ void __launch_bounds__(1024) k_bin_scan(const int32_t* __restrict__ count,
                                                   int32_t* __restrict__ off, int32_t P) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t b = 0; b < P; b += 1024) {
    const int32_t i = b + (int32_t)threadIdx.x;
    const int32_t c = i < P ? count[i] : 0;
    int32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int32_t t = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += v;
      }
      wsum[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int32_t before = carry + (wid ? wsum[wid - 1] : 0) + incl - c;
    if (i < P) off[i] = before;
    __syncthreads();
    if (threadIdx.x == 1023) carry = before + c;
    __syncthreads();
  }
}

// Patch bins, step 3: item i goes to position off[patch] + rank.
__global__ void __launch_bounds__(256) k_bin_scatter(K3Queues Q) {
  const int64_t n = (int64_t)min(*Q.n_count, Q.cap);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int2 k = Q.nkey[i];
    const int64_t pos = (int64_t)__ldg(Q.bin_off + k.x) + k.y;
    if (pos < n) Q.perm[pos] = (int32_t)i;
  }
}

// Newton pass in patch order (scenes beyond the shared-memory patch table).
// A batch of 32 items taken through `perm` holds one patch (two where a bin
// ends): the warp stages that patch's 48 power coefficients in its own
// shared-memory slot and every lane re-reads them as broadcasts each iteration
// (no per-lane coefficient registers, no 32-line L1 gathers: ncu put
// k3_newton<false> at 99% L1/LSU and 15% FP64 pipe at config 5).  Items of one
// query are no longer adjacent, so chi / flags go out as one atomic per root.
#ifndef GWN_NEWTON_MINB_BIN
#define GWN_NEWTON_MINB_BIN 5
#endif
#ifndef GWN_NB_PREFETCH
#define GWN_NB_PREFETCH 1
#endif
#ifndef GWN_NB_RUN
#define GWN_NB_RUN 8
#endif
// A warp reserves a run of up to GWN_NB_RUN consecutive batches at a time, so
// its shared-memory table stays valid from batch to batch (the coefficient
// load that fills it is a full L2 round trip on the batch's critical path:
// 29% of the stall samples when every batch re-staged its patch).
__global__ void __launch_bounds__(128, GWN_NEWTON_MINB_BIN)
k3_newton_binned(WaveArgs w, const int32_t* __restrict__ perm) {
  __shared__ __align__(16) double wtab[4][48];
  const int64_t n = (int64_t)min(*w.n_count, w.n_cap);
  const int64_t nb = (n + 31) >> 5;  // batches
  const int64_t nwarps = (int64_t)gridDim.x * 4;
  // run length: long runs for table reuse, short ones when there is little work
  const int64_t R = max((int64_t)1, min((int64_t)GWN_NB_RUN, nb / (nwarps * 4)));
  unsigned long long iters = 0, roots = 0;
  const int lane = threadIdx.x & 31;
  double* tab = wtab[threadIdx.x >> 5];
  unsigned r_cur = 0, r_nxt = 0;
  if (lane == 0) {
    r_cur = reserve_batch(w.n_work);
    r_nxt = reserve_batch(w.n_work);
  }
  int64_t b = R * (int64_t)__shfl_sync(0xffffffffu, r_cur, 0);  // current batch
  int64_t run_end = b + R;
  int32_t cur_p = -1;
#if GWN_NB_PREFETCH
  // perm index two batches ahead, item lines prefetched one batch ahead
  int32_t idx = b * 32 + lane < n ? perm[b * 32 + lane] : -1;
#else
  NewtonItem it{};
  if (b * 32 + lane < n) it = w.nq[perm[b * 32 + lane]];
#endif
  while (b < nb) {
    // the batch after this one: next of the run, else the next run's first
    int64_t b2 = b + 1, run_end2 = run_end;
    if (b2 >= run_end) {
      b2 = R * (int64_t)__shfl_sync(0xffffffffu, r_nxt, 0);
      run_end2 = b2 + R;
      if (lane == 0 && b2 < nb) r_nxt = reserve_batch(w.n_work);
    }
#if GWN_NB_PREFETCH
    const int32_t idx2 = b2 * 32 + lane < n ? perm[b2 * 32 + lane] : -1;
    NewtonItem it{};
    if (idx >= 0) it = w.nq[idx];
    const bool have = idx >= 0;
#else
    NewtonItem nx{};
    if (b2 * 32 + lane < n) nx = w.nq[perm[b2 * 32 + lane]];
    const bool have = b * 32 + lane < n;
#endif
    int32_t chi = 0, fl = 0;
    unsigned rem = __ballot_sync(0xffffffffu, have);
    while (rem) {
      const int leader = __ffs(rem) - 1;
      const int32_t p = __shfl_sync(0xffffffffu, it.patch, leader);
      const bool mine = have && it.patch == p;
      rem &= ~__ballot_sync(0xffffffffu, mine);
      if (p != cur_p) {
        __syncwarp();
        if (lane < 24)
          reinterpret_cast<double2*>(tab)[lane] =
              __ldg(reinterpret_cast<const double2*>(w.powc + 48 * (int64_t)p) + lane);
        __syncwarp();
        cur_p = p;
      }
#if GWN_NB_PREFETCH
      // the next batch's item lines into L1 while this one is solved
      if (idx2 >= 0 && !rem)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(w.nq + idx2));
#endif
      if (mine) {
        const RootResult r = newton_solve_pow<2>(tab, it.qa, it.qb, it.qc, it.u, it.v, w.prm);
        newton_own(w, it.slot, it.code, r, chi, fl, iters, roots);
      }
    }
    if (chi) atomicAdd(&w.chi[it.slot], chi);
    if (fl) atomicOr(&w.flags[it.slot], fl);
#if GWN_NB_PREFETCH
    idx = idx2;
#else
    it = nx;
#endif
    b = b2;
    run_end = run_end2;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see k3_newton
  warp_sum_u64(&w.counters[CNT_NEWTON], iters);
  warp_sum_u64(&w.counters[CNT_ROOTS], roots);
}

static int grid_for(const void* fn, int sm_count, int block = 128, size_t smem = 0) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem);
  if (per_sm < 1) per_sm = 1;
  return sm_count * per_sm;
}

// K3 driver: candidate tests, then the fallback on a side stream
// concurrently with the Newton pass; every kernel reads its queue length
// from device memory -- no host synchronisation.
cudaError_t launch_intersect(const gwn_scene* sc, const Round& rd, const K3Queues& Q,
                             const unsigned long long* npairs_dev, const double* qproj,
                             int32_t* chi, int32_t* flags, unsigned long long* counters,
                             unsigned long long* newton_work, cudaEvent_t* ev4,
                             cudaEvent_t* join, const RecordSink* rec, cudaStream_t st) {
  static thread_local int g_cand = 0, g_fb = 0, g_newton = 0, g_newton_s = 0, g_newton_b = 0,
                          g_dev = -1;
  if (g_dev != sc->device) {
    g_cand = grid_for((const void*)k3_candidates, sc->sm_count, kCandBlock);
    // fallback: 3 blocks per SM spread its few, long-lived items thinly
    // (measured on config 2 against 1, 2, 4, 6, 8)
    g_fb = sc->sm_count * 3;
    // Newton at full occupancy: its dynamic fetch drains the queue, then the
    // fallback blocks take the SMs
    g_newton = grid_for((const void*)k3_newton<false>, sc->sm_count);
    g_newton_s = grid_for((const void*)k3_newton<true>, sc->sm_count, 128,
                          sizeof(double) * kTabStride * kTabMaxP);
    g_newton_b = grid_for((const void*)k3_newton_binned, sc->sm_count);
    g_dev = sc->device;
  }
  cudaError_t e = cudaSuccess;
  WaveArgs w{rd.leaves, qproj, rd.proj, rd.powc, sc->dprm, chi, flags,
             rec ? rec->rec : nullptr, rec ? rec->count : nullptr, rec ? rec->cap : 0ull,
             counters, Q.overflow, Q.nq, Q.n_count, Q.cap, newton_work,
             rd.sub_offs, rd.sub, rd.subbox, rd.subskip, rd.subgc, rd.sub_level};
  const bool binned = Q.n_bins > 0;
  if (binned &&
      (e = cudaMemsetAsync(Q.bin_count, 0, sizeof(int32_t) * Q.n_bins, st)) != cudaSuccess)
    return e;
  if (ev4) cudaEventRecord(ev4[0], st);
  tl_mark(st, "k3 start");
  static const bool pdl_cand = [] {
    const char* e = getenv("GWN_PDL");
    return !(e && atoi(e) == 0);
  }();
  if (pdl_cand && !ev4) {  // programmatic dependent launch behind the cull
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g_cand);
    cfg.blockDim = dim3(kCandBlock);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if ((e = cudaLaunchKernelEx(&cfg, k3_candidates, npairs_dev, Q, w)) != cudaSuccess) return e;
  } else {
    k3_candidates<<<g_cand, kCandBlock, 0, st>>>(npairs_dev, Q, w);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // The fallback (few, latency-bound items) runs on a side stream,
  // concurrently with the Newton pass and K4; the engine joins it (`join`)
  // before K5 reads the accumulators.
  // per host thread and device (streams and events belong to one device)
  static thread_local cudaStream_t t_side[64] = {};
  static thread_local cudaEvent_t t_fork[64] = {}, t_join[64] = {};
  cudaStream_t& side = t_side[sc->device & 63];
  cudaEvent_t& fork_ev = t_fork[sc->device & 63];
  cudaEvent_t& join_ev = t_join[sc->device & 63];
  if (!side) {
    // high priority: the fallback's blocks are dispatched ahead of the Newton
    // pass's, so its long dependent chains start first
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    const int prio = hi_prio;
    if ((e = cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, prio)) != cudaSuccess)
      return e;
    if ((e = cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  // In timing mode (ev4) everything runs on `st` so each kernel's events
  // measure it alone.  GWN_PDL (default on): the fallback runs on `st` too and
  // the Newton pass is a programmatic dependent launch behind it, so the
  // fallback's few long-lived blocks are resident first and Newton fills the
  // rest of the GPU concurrently (no side stream, no join).
  static const bool pdl = [] {
    const char* e = getenv("GWN_PDL");
    return !(e && atoi(e) == 0);
  }();
  // (patch-bin scenes: the scan and scatter sit between the fallback and the
  // Newton pass, so there is no programmatic pair to form; the fallback goes
  // to the high-priority side stream and overlaps the Newton pass and K4)
  const bool use_pdl = pdl && !ev4 && !binned;
  cudaStream_t fs = (ev4 || use_pdl) ? st : side;
  if (!ev4 && !use_pdl) {
    if ((e = cudaEventRecord(fork_ev, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(side, fork_ev, 0)) != cudaSuccess) return e;
  }
  if (ev4) cudaEventRecord(ev4[1], fs);
  tl_mark(fs, "fb start");
  k3_fallback<<<g_fb, 32 * kFbWarps, 0, fs>>>(Q.fq, Q.f_count, w);
  tl_mark(fs, "fb done");
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (ev4) cudaEventRecord(ev4[2], fs);
  if (!ev4 && !use_pdl) {
    if ((e = cudaEventRecord(join_ev, side)) != cudaSuccess) return e;
    *join = join_ev;
  }
  tl_mark(st, "newton start");
  static const bool smem_ok = [] {
    const char* e = getenv("GWN_NEWTON_SMEM");
    return !(e && atoi(e) == 0);
  }();
  const bool tabled = smem_ok && sc->P <= kTabMaxP;
  if (binned) {  // items in patch order (the fallback runs meanwhile)
    k_bin_scan<<<1, 1024, 0, st>>>(Q.bin_count, Q.bin_off, Q.n_bins);
    k_bin_scatter<<<sc->sm_count * 8, 256, 0, st>>>(Q);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // (stage timing: ev4[2] -> ev4[4] is the bin scan and scatter, which the
  // engine books with the candidate test -- together they build the Newton
  // queue; ev4[4] -> ev4[3] is the Newton kernel alone)
  if (ev4) cudaEventRecord(ev4[4], st);
  if (binned) {
    // (a plain launch: the scan and scatter above sit between the fallback and
    // this kernel, so there is no programmatic pair to form)
    k3_newton_binned<<<g_newton_b, 128, 0, st>>>(w, Q.perm);
  } else if (use_pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tabled ? g_newton_s : g_newton);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = tabled ? sizeof(double) * kTabStride * sc->P : 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int32_t P32 = (int32_t)sc->P;
    e = tabled ? cudaLaunchKernelEx(&cfg, k3_newton<true>, w, P32)
               : cudaLaunchKernelEx(&cfg, k3_newton<false>, w, P32);
    if (e != cudaSuccess) return e;
  } else if (tabled) {
    k3_newton<true><<<g_newton_s, 128, sizeof(double) * kTabStride * sc->P, st>>>(w, (int32_t)sc->P);
  } else {
    k3_newton<false><<<g_newton, 128, 0, st>>>(w, (int32_t)sc->P);
  }
  tl_mark(st, "newton done");
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (ev4) cudaEventRecord(ev4[3], st);
  return e;
}

K3Queues k3_queues(void* scratch, int64_t cap, unsigned long long* k3cnt, int64_t P) {
  char* p = (char*)scratch;
  K3Queues q;
  auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };  // keep every queue aligned
  q.pairs = (int2*)p;
  p += up(sizeof(int2) * cap);
  q.fq = (NodeItem*)p;
  p += up(sizeof(NodeItem) * cap);
  q.nq = (NewtonItem*)p;
#ifndef GWN_NEWTON_BIN
#define GWN_NEWTON_BIN 1
#endif
  // GWN_NEWTON_BIN=0 (environment, tests): the unbinned Newton pass
  static const bool bin_ok = [] {
    const char* e = getenv("GWN_NEWTON_BIN");
    return !(e && atoi(e) == 0);
  }();
  if (GWN_NEWTON_BIN && bin_ok && P > kTabMaxP && cap < (1ll << 31)) {
    p += up(sizeof(NewtonItem) * cap);
    q.nkey = (int2*)p;
    p += up(sizeof(int2) * cap);
    q.perm = (int32_t*)p;
    p += up(sizeof(int32_t) * cap);
    q.bin_count = (int32_t*)p;
    p += up(sizeof(int32_t) * P);
    q.bin_off = (int32_t*)p;
    q.n_bins = (int32_t)P;
  }
  q.f_count = k3cnt;
  q.n_count = k3cnt + 1;
  q.overflow = (int*)(k3cnt + 2);
  q.cap = (unsigned long long)cap;
  return q;
}

// (sized for the bins whether or not this round uses them)
size_t intersect_scratch_bytes(int64_t pair_cap, int64_t P) {
  size_t b = (sizeof(int2) + sizeof(NodeItem) + sizeof(NewtonItem)) * pair_cap + 1024;
  if (P > kTabMaxP) b += (sizeof(int2) + sizeof(int32_t)) * pair_cap + 2 * sizeof(int32_t) * P + 1024;
  return b;
}

}  // namespace gwn
