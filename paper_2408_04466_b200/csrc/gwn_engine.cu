// gwn_engine.cu -- the batched engine (SPEC.md:371-380 winding_number, for
// many queries) and the C-ABI entry points that need device work.
//
// Per chunk of queries, per direction round r (all active queries of a round
// share d_r, so the patch hierarchy of the round is shared):
//   K2 cull count -> exclusive scan -> K2 fill   (candidate pairs by query)
//   K3 intersect + segmented warp reduction       (chi, flags per query)
//   K4 boundary term                              (B, flags per query)
//   K5 finalize: w = chi + B, or jitter / re-shoot
// Re-shot queries are compacted into the next round's active list.
#include <cub/cub.cuh>

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "gwn_internal.h"
#include "gwn_k3.cuh"

namespace gwn {

// w = chi + (sum of the chunk partial angles) / 2 pi, rounded the same way in
// every finalize path (explicit roundings: no FMA contraction choices)
__device__ __forceinline__ double w_of(int32_t chi, double ang) {
  return __dadd_rn((double)chi, __dmul_rn(ang, 0.15915494309189533576888));
}

// K5 for one query slot s (query q): done / jitter / re-shoot; returns true
// when q goes to the next round.
__device__ __forceinline__ bool finalize_one(
    int32_t s, int32_t q, int32_t m, int32_t f, double w, int round, int max_rounds,
    int max_jitters, uint64_t seed, int64_t index_base, const int64_t* __restrict__ qidx,
    double jscale, const double* __restrict__ q0, double* __restrict__ pos,
    int8_t* __restrict__ jit, int8_t* __restrict__ jreason, double* __restrict__ w_out,
    int8_t* __restrict__ st_out) {
  bool push = false;
  if (f & (FLAG_ONSURF | FLAG_DEGEN)) {
    int reason = (f & FLAG_ONSURF) ? GWN_STATUS_ON_SURFACE : GWN_STATUS_DEGENERATE;
    int j = round > 0 ? jit[q] : 0;  // round 0: jit / pos not yet initialised
    if (j < max_jitters && round + 1 >= max_rounds) {
      w_out[q] = w;  // jitter budget left but no round to use it (oracle eval_query)
      st_out[q] = GWN_STATUS_EXHAUSTED;
    } else if (j < max_jitters) {
      ++j;
      jit[q] = (int8_t)j;
      jreason[q] = (int8_t)reason;
      // deterministic jitter (same hash as gwn_jitter_dir / the oracle)
      uint64_t st = seed ^ 0x5851F42D4C957F2Dull;
      st ^= (uint64_t)(qidx ? qidx[q] : index_base + q) * 0x9E3779B97F4A7C15ull;
      st ^= (uint64_t)(j + 1) * 0xC2B2AE3D27D4EB4Full;
      double v[3];
      for (int k = 0; k < 3; ++k) {
        uint64_t z = (st += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        v[k] = __dadd_rn(__dmul_rn(2.0, __dmul_rn((double)(z >> 11), 1.0 / 9007199254740992.0)),
                         -1.0);
      }
      double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                      __dmul_rn(v[2], v[2])));
      if (n < 1e-3) {
        v[0] = 1.0; v[1] = 0.0; v[2] = 0.0;
      } else {
        for (int k = 0; k < 3; ++k) v[k] = __ddiv_rn(v[k], n);
      }
      for (int k = 0; k < 3; ++k)
        pos[3 * (int64_t)q + k] = __dadd_rn(q0[3 * (int64_t)q + k], __dmul_rn(jscale, v[k]));
      push = true;
    } else {
      w_out[q] = w;  // still on the surface / boundary after max_jitters
      st_out[q] = GWN_STATUS_JITTER_EXHAUSTED;
    }
  } else if (f & (FLAG_RESHOOT | FLAG_BAND)) {
    if (round + 1 < max_rounds) {
      push = true;
      if (round == 0) {  // next round reads pos / jit of the queries it gets
        jit[q] = 0;
        for (int k = 0; k < 3; ++k) pos[3 * (int64_t)q + k] = q0[3 * (int64_t)q + k];
      }
    } else {
      w_out[q] = w;
      st_out[q] = GWN_STATUS_EXHAUSTED;
    }
  } else {
    w_out[q] = w;
    st_out[q] = (round > 0 && jit[q]) ? jreason[q] : (int8_t)GWN_STATUS_OK;
  }
  return push;
}

// Last block of a K5 launch: copy the round's scalar block (eval counters
// and round scalars) into mapped pinned host memory -- the host's one round
// trip per round reads it after the stream sync, no D2H copy op.
// The last block's first (nblk+1)/2 threads each move one 16-byte pair:
// parallel PCIe writes (a single thread writing the values one by one, then
// a system fence, cost ~5 us per round at config 2).  `host` holds
// nblk + 1 values, `blk` is readable one past its end (workspace padding).
__device__ __forceinline__ void publish_scalars(unsigned long long* __restrict__ done,
                                                const unsigned long long* __restrict__ blk,
                                                unsigned long long* __restrict__ host, int nblk) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long prev = atomicAdd(done, 1ull);
    s_last = prev == (unsigned long long)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && (int)threadIdx.x < (nblk + 1) / 2) {
    __threadfence();
    const int k = 2 * threadIdx.x;
    ulonglong2 v;
    v.x = *(volatile const unsigned long long*)(blk + k);
    v.y = *(volatile const unsigned long long*)(blk + k + 1);
    reinterpret_cast<ulonglong2*>(host)[threadIdx.x] = v;
    // no system fence: the host reads only after synchronising the stream,
    // and kernel completion orders these writes before it
  }
}

// K5: per active query decide done / jitter / re-shoot.
__device__ __forceinline__ void finalize_body(int32_t m, const int32_t* __restrict__ active,
                           const int32_t* __restrict__ chi, const int32_t* __restrict__ flags,
                           const double* __restrict__ bpart, int nchunk, int round, int max_rounds,
                           int max_jitters, uint64_t seed, int64_t index_base,
                           const int64_t* __restrict__ qidx, double jscale,
                           const double* __restrict__ q0, double* __restrict__ pos,
                           int8_t* __restrict__ jit, int8_t* __restrict__ jreason,
                           double* __restrict__ w_out, int8_t* __restrict__ st_out,
                           int32_t* __restrict__ next, int32_t* __restrict__ next_n,
                           const unsigned long long* __restrict__ pair_count,
                           unsigned long long pair_cap) {
  int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  bool push = false;
  int32_t q = 0;
  // candidate buffer overflowed: the round is re-run (nothing written)
  if (s < m && *pair_count <= pair_cap) {
    q = active ? active[s] : s;
    const int32_t f = flags[s];
    // boundary term: per-chunk partial angles summed in chunk order
    // (deterministic), (2 * angle) / (4 pi)
    double ang = 0.0;
    for (int c = 0; c < nchunk; ++c) ang = __dadd_rn(ang, bpart[(int64_t)c * m + s]);
    const double w = w_of(chi[s], ang);
    push = finalize_one(s, q, m, f, w, round, max_rounds, max_jitters, seed, index_base, qidx,
                        jscale, q0, pos, jit, jreason, w_out, st_out);
  }
  // warp-aggregated compaction of the re-shot queries
  unsigned mask = __ballot_sync(0xffffffffu, push);
  if (mask) {
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    int32_t base = 0;
    if (lane == leader) base = atomicAdd(next_n, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (push) next[base + __popc(mask & ((1u << lane) - 1))] = q;
  }
}

__global__ void k_finalize(int32_t m, const int32_t* __restrict__ active,
                           const int32_t* __restrict__ chi, const int32_t* __restrict__ flags,
                           const double* __restrict__ bpart, int nchunk, int round, int max_rounds,
                           int max_jitters, uint64_t seed, int64_t index_base,
                           const int64_t* __restrict__ qidx, double jscale,
                           const double* __restrict__ q0, double* __restrict__ pos,
                           int8_t* __restrict__ jit, int8_t* __restrict__ jreason,
                           double* __restrict__ w_out, int8_t* __restrict__ st_out,
                           int32_t* __restrict__ next, int32_t* __restrict__ next_n,
                           const unsigned long long* __restrict__ pair_count,
                           unsigned long long pair_cap, unsigned long long* done,
                           const unsigned long long* blk, unsigned long long* host, int nblk) {
  finalize_body(m, active, chi, flags, bpart, nchunk, round, max_rounds, max_jitters, seed,
                index_base, qidx, jscale, q0, pos, jit, jreason, w_out, st_out, next, next_n,
                pair_count, pair_cap);
  publish_scalars(done, blk, host, nblk);
}

__device__ __forceinline__ void finalize4_group(int32_t s0, int32_t m,
                            const int32_t* __restrict__ chi,
                            const int32_t* __restrict__ flags, const double* __restrict__ bpart,
                            int nchunk, int max_rounds, int max_jitters, uint64_t seed,
                            int64_t index_base, const int64_t* __restrict__ qidx, double jscale,
                            const double* __restrict__ q0, double* __restrict__ pos,
                            int8_t* __restrict__ jit, int8_t* __restrict__ jreason,
                            double* __restrict__ w_out, int8_t* __restrict__ st_out,
                            int32_t* __restrict__ next, int32_t* __restrict__ next_n, bool ovf);

// K5, round 0 with the identity slot map (the common case): four queries per
// thread with 16-byte loads of chi / flags / partials and 16- and 4-byte
// stores of w / status; flagged queries (rare) take finalize_one and a plain
// atomic append.
__device__ __forceinline__ void finalize4_body(int32_t m, const int32_t* __restrict__ chi,
                            const int32_t* __restrict__ flags, const double* __restrict__ bpart,
                            int nchunk, int max_rounds, int max_jitters, uint64_t seed,
                            int64_t index_base, const int64_t* __restrict__ qidx, double jscale,
                            const double* __restrict__ q0, double* __restrict__ pos,
                            int8_t* __restrict__ jit, int8_t* __restrict__ jreason,
                            double* __restrict__ w_out, int8_t* __restrict__ st_out,
                            int32_t* __restrict__ next, int32_t* __restrict__ next_n,
                            const unsigned long long* __restrict__ pair_count,
                            unsigned long long pair_cap) {
  // the round is re-run if the candidate buffer overflowed; the flag is tested
  // after each group's loads are issued, so its round trip overlaps them
  const bool ovf = *pair_count > pair_cap;
  // grid-stride over groups of four: a few blocks per SM keep the
  // publish_scalars completion counter (one atomic per block) short
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 4 * g < m;
       g += (int64_t)gridDim.x * blockDim.x)
    finalize4_group((int32_t)(4 * g), m, chi, flags, bpart, nchunk, max_rounds, max_jitters,
                    seed, index_base, qidx, jscale, q0, pos, jit, jreason, w_out, st_out, next,
                    next_n, ovf);
}

__device__ __forceinline__ void finalize4_group(int32_t s0, int32_t m,
                            const int32_t* __restrict__ chi,
                            const int32_t* __restrict__ flags, const double* __restrict__ bpart,
                            int nchunk, int max_rounds, int max_jitters, uint64_t seed,
                            int64_t index_base, const int64_t* __restrict__ qidx, double jscale,
                            const double* __restrict__ q0, double* __restrict__ pos,
                            int8_t* __restrict__ jit, int8_t* __restrict__ jreason,
                            double* __restrict__ w_out, int8_t* __restrict__ st_out,
                            int32_t* __restrict__ next, int32_t* __restrict__ next_n,
                            bool ovf) {
  if (s0 + 4 > m) {  // ragged tail: scalar
    if (ovf) return;
    for (int32_t s = s0; s < m; ++s) {
      double ang = 0.0;
      for (int c = 0; c < nchunk; ++c) ang = __dadd_rn(ang, bpart[(int64_t)c * m + s]);
      const double w = w_of(chi[s], ang);
      if (finalize_one(s, s, m, flags[s], w, 0, max_rounds, max_jitters, seed, index_base, qidx,
                       jscale, q0, pos, jit, jreason, w_out, st_out))
        next[atomicAdd(next_n, 1)] = s;
    }
    return;
  }
  // volatile loads: issued here, before the overflow test below
  int4 c4, f4;
  asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(c4.x), "=r"(c4.y), "=r"(c4.z), "=r"(c4.w) : "l"(chi + s0));
  asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(f4.x), "=r"(f4.y), "=r"(f4.z), "=r"(f4.w) : "l"(flags + s0));
  if (ovf) return;
  double ang[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c = 0; c < nchunk; ++c) {
    const double* b = bpart + (int64_t)c * m + s0;
    if ((m & 1) == 0) {
      const double2 x = *reinterpret_cast<const double2*>(b);
      const double2 y = *reinterpret_cast<const double2*>(b + 2);
      ang[0] = __dadd_rn(ang[0], x.x); ang[1] = __dadd_rn(ang[1], x.y);
      ang[2] = __dadd_rn(ang[2], y.x); ang[3] = __dadd_rn(ang[3], y.y);
    } else {
      for (int k = 0; k < 4; ++k) ang[k] = __dadd_rn(ang[k], b[k]);
    }
  }
  const int cc[4] = {c4.x, c4.y, c4.z, c4.w};
  const int ff[4] = {f4.x, f4.y, f4.z, f4.w};
  double w[4];
  for (int k = 0; k < 4; ++k) w[k] = w_of(cc[k], ang[k]);
  if ((ff[0] | ff[1] | ff[2] | ff[3]) == 0) {
    *reinterpret_cast<double2*>(w_out + s0) = make_double2(w[0], w[1]);
    *reinterpret_cast<double2*>(w_out + s0 + 2) = make_double2(w[2], w[3]);
    *reinterpret_cast<int32_t*>(st_out + s0) = 0;  // 4 x GWN_STATUS_OK
    return;
  }
  for (int k = 0; k < 4; ++k) {
    const int32_t s = s0 + k;
    if (finalize_one(s, s, m, ff[k], w[k], 0, max_rounds, max_jitters, seed, index_base, qidx,
                     jscale, q0, pos, jit, jreason, w_out, st_out))
      next[atomicAdd(next_n, 1)] = s;
  }
}

__global__ void k_finalize4(int32_t m, const int32_t* __restrict__ chi,
                            const int32_t* __restrict__ flags, const double* __restrict__ bpart,
                            int nchunk, int max_rounds, int max_jitters, uint64_t seed,
                            int64_t index_base, const int64_t* __restrict__ qidx, double jscale,
                            const double* __restrict__ q0, double* __restrict__ pos,
                            int8_t* __restrict__ jit, int8_t* __restrict__ jreason,
                            double* __restrict__ w_out, int8_t* __restrict__ st_out,
                            int32_t* __restrict__ next, int32_t* __restrict__ next_n,
                            const unsigned long long* __restrict__ pair_count,
                            unsigned long long pair_cap, unsigned long long* done,
                            const unsigned long long* blk, unsigned long long* host, int nblk) {
  finalize4_body(m, chi, flags, bpart, nchunk, max_rounds, max_jitters, seed, index_base, qidx,
                 jscale, q0, pos, jit, jreason, w_out, st_out, next, next_n, pair_count,
                 pair_cap);
  publish_scalars(done, blk, host, nblk);
}

// GWN_TRACE=1: host wall-clock trace of the eval phases (development aid)
thread_local GpuTimeline* g_tl = nullptr;

struct Trace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  Trace() : on(getenv("GWN_TRACE") != nullptr) { t0 = last = std::chrono::steady_clock::now(); }
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[gwn] %-28s +%8.1f us  (%8.1f)\n", what,
            std::chrono::duration<double, std::micro>(now - last).count(),
            std::chrono::duration<double, std::micro>(now - t0).count());
    last = now;
  }
};

// Per-thread, per-device eval workspace: one block carved by a bump
// allocator and kept across evals.  gwn_eval synchronises its streams before
// returning, so the next eval on the same thread may reuse the block; evals
// on other threads have their own.  Requests past the block fall back to
// stream-ordered allocations for this eval, and the block grows to the
// high-water mark at the next one.  (One allocation per eval instead of
// ~14: the host reaches the first kernel launch ~10 us sooner.)
struct WsCache {
  char* buf = nullptr;
  size_t cap = 0, want = 0;
  void* k3 = nullptr;  // K3 queue scratch, kept the same way
  size_t k3_cap = 0;
};
static thread_local WsCache t_wscache[64];

void release_boundary_caches(int device);  // gwn_boundary.cu

// this host thread's eval workspace on `device` (gwn_release_caches)
static void release_ws_cache(int device) {
  WsCache& c = t_wscache[device & 63];
  if (c.buf) cudaFree(c.buf);
  if (c.k3) cudaFree(c.k3);
  c = WsCache();
  release_boundary_caches(device);
}

struct Workspace {
  cudaStream_t st;
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  WsCache* c = nullptr;
  size_t off = 0;
  void begin(int device) {
    c = &t_wscache[device & 63];
    if (c->want > c->cap) {
      if (c->buf) cudaFreeAsync(c->buf, st);
      c->buf = nullptr;
      c->cap = 0;
      const size_t want = c->want + c->want / 4;
      if (cudaMallocAsync((void**)&c->buf, want, st) == cudaSuccess) {
        c->cap = want;
      } else {
        c->buf = nullptr;
        cudaGetLastError();  // fall back to per-request allocations
      }
    }
  }
  template <class T>
  T* get(size_t n) {
    if (err != cudaSuccess) return nullptr;
    const size_t bytes = (n * sizeof(T) + 16 + 255) & ~(size_t)255;
    off += bytes;
    if (c) c->want = std::max(c->want, off);
    if (c && c->buf && off <= c->cap) return (T*)(c->buf + off - bytes);
    void* p = nullptr;
    err = cudaMallocAsync(&p, bytes, st);
    if (err == cudaSuccess) ptrs.push_back(p);
    return (T*)p;
  }
  // K3 scratch of at least `bytes` (cached; grows stream-ordered)
  cudaError_t k3(size_t bytes, void** out) {
    if (c->k3_cap < bytes) {
      if (c->k3) cudaFreeAsync(c->k3, st);
      c->k3 = nullptr;
      c->k3_cap = 0;
      const cudaError_t e = cudaMallocAsync(&c->k3, bytes, st);
      if (e != cudaSuccess) return e;
      c->k3_cap = bytes;
    }
    *out = c->k3;
    return cudaSuccess;
  }
  void release() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    ptrs.clear();
  }
};

}  // namespace gwn

using namespace gwn;

// gwn_release_caches: this host thread's eval workspace on `device` (the
// buffers grow to the largest batch seen and are kept for the next eval)
extern "C" int gwn_release_caches(int device) {
  if (device < 0) {
    set_error("gwn_release_caches: invalid device");
    return GWN_E_INVALID;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  release_ws_cache(device);
  cudaDeviceSynchronize();
  cudaSetDevice(cur);
  return GWN_OK;
}

#define CKE(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      set_error("%s failed: %s", #call, cudaGetErrorString(e_));              \
      rc = (e_ == cudaErrorMemoryAllocation) ? GWN_E_OOM : GWN_E_CUDA;         \
      goto done;                                                               \
    }                                                                          \
  } while (0)

// Round r of the scene (built on first use); the pointer stays valid for
// the scene's lifetime (deque), taken under the scene mutex.
static cudaError_t ensure_round(gwn_scene* sc, int r, cudaStream_t st, const Round** out,
                                double* ms_build = nullptr) {
  std::lock_guard<std::mutex> lk(sc->mu);
  if ((int)sc->rounds.size() <= r) {
    const auto t0 = std::chrono::steady_clock::now();
    const cudaError_t e = build_round(sc, r, st);
    if (e != cudaSuccess) return e;
    if (ms_build)
      *ms_build += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count();
  }
  *out = &sc->rounds[r];
  return cudaSuccess;
}

static int eval_core(gwn_scene* sc, const double* queries, int64_t n, int64_t index_base,
                     const int64_t* qidx, double* w_out, int8_t* status_out, int32_t flags,
                     void* stream) {
  int rc = GWN_OK;
  if (!sc || n < 0 || (n > 0 && (!queries || !w_out || !status_out))) {
    set_error("gwn_eval: invalid arguments");
    return GWN_E_INVALID;
  }
  if (n == 0) return GWN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Trace tr;
  GpuTimeline tl;
  Workspace ws;
  // rounds past the scene's cache (prm.cached_rounds, default 4: round 0
  // with the far field's local expansions and the first re-shoot rounds,
  // which every large batch needs): built for this eval in
  // `spill` (one at a time) and freed at its end, so a batch of stubborn
  // queries re-shot up to 32 times cannot pile 32 full-scene rounds on the
  // device (~5 GB each at config 5)
  Round spill;
  int spill_r = -1;
  ws.st = st;
  const bool host = (flags & GWN_HOST_BUFFERS) != 0;
  // auto chunk: 4M queries (2M when the boundary partials are wide; 32M for
  // far-field scenes: a local-expansion leaf's queries share one warp's list
  // only when the leaves are well filled, and every chunk pays the re-shoot
  // rounds' latency -- config 5 at 2^26 queries: 1071 ms in 8M chunks, 958 in
  // 32M, 930 in one 64M chunk, whose K3 queues alone take ~60 GB)
  const int64_t chunk_max = sc->prm.chunk_queries > 0 ? sc->prm.chunk_queries
                            : sc->ff_n > 0               ? (1ll << 25)
                            : boundary_chunks(sc, 0) > 16 ? (1ll << 21)
                                                          : (1ll << 22);
  // device scalar block, published to mapped pinned memory once per round
  // by K5's last block:
  // [0, CNT_N) eval counters, CNT_N + [0] candidate count, [1] next active
  // count, [2] K5 blocks done, [4] fallback items, [5] Newton items, [6] overflow,
  // [7] Newton work
  constexpr int kBlk = CNT_N + 8;
  int64_t* h_scalar = nullptr;
  unsigned long long* h_map = nullptr;  // device view of h_scalar (mapped)
  const double* d_q = queries;
  double* d_w = w_out;
  int8_t* d_st = status_out;
  gwn_stats stats;
  memset(&stats, 0, sizeof stats);
  stats.queries = n;
  cudaEvent_t ev[8] = {}, ev4[5] = {}, evb[3] = {};
  int64_t launches = 0;
  // host buffers, large batches: chunks pipelined against the copies
  // (H2D of chunk k+1 and D2H of chunk k-1 overlap chunk k's rounds)
  const bool pipe = host && n >= (1ll << 18) && !sc->timed;
  // copy streams per host thread AND device (a stream belongs to the device
  // current at its creation)
  static thread_local cudaStream_t t_cs_in[64] = {}, t_cs_out[64] = {};
  cudaStream_t& cs_in = t_cs_in[sc->device & 63];
  cudaStream_t& cs_out = t_cs_out[sc->device & 63];
  std::vector<cudaEvent_t> pev;  // per chunk: [2k] input copied, [2k+1] chunk done
  unsigned long long* d_cnt = nullptr;
  unsigned long long h_cnt[CNT_N];
  CKE(cudaSetDevice(sc->device));
  {
    // pinned round scalars: one small buffer per host thread (gwn_eval
    // synchronises its stream before returning, so reuse is safe)
    static thread_local int64_t* t_pinned = nullptr;
    static thread_local unsigned long long* t_map = nullptr;
    if (!t_pinned) {
      // portable: one host thread may drive several devices (UVA gives the
      // same device view on each)
      CKE(cudaHostAlloc(&t_pinned, (kBlk + 1) * sizeof(int64_t),
                        cudaHostAllocMapped | cudaHostAllocPortable));
      CKE(cudaHostGetDevicePointer((void**)&t_map, t_pinned, 0));
    }
    h_scalar = t_pinned;
    h_map = t_map;
  }
  g_tl = getenv("GWN_TIMELINE") ? &tl : nullptr;
  tl_mark(st, "start");
  tr.mark("setup");
  ws.begin(sc->device);
  d_cnt = ws.get<unsigned long long>(kBlk);
  CKE(ws.err);
  if (host) {
    double* dq = ws.get<double>((size_t)(3 * n));
    d_w = ws.get<double>((size_t)n);
    d_st = ws.get<int8_t>((size_t)n);
    CKE(ws.err);
    if (!pipe)
      CKE(cudaMemcpyAsync(dq, queries, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    d_q = dq;
  }
  if (sc->timed) {
    for (auto& e : ev) CKE(cudaEventCreate(&e));
    for (auto& e : ev4) CKE(cudaEventCreate(&e));
    for (auto& e : evb) CKE(cudaEventCreate(&e));
  }
  {
    int64_t cm = n < chunk_max ? n : chunk_max;
    std::vector<int64_t> cst{0};  // chunk starts
    if (pipe) {
      // parts: measured at config 2 (2^20 queries, pinned host buffers), e2e
      // G q/s: 2 chunks 1.63, 4 1.70, 6 1.79, 8 1.55, 12 1.27 (splitting the
      // last chunk or issuing every input copy up front did not help);
      // far-field scenes: three (their steps are long next to the copies, and
      // larger chunks keep the local-expansion leaves' warps uniform; config 5
      // at 2^26 queries: 2 chunks 323.1 ms, 3 320.0, 4 321.6)
#ifndef GWN_PIPE_FF
#define GWN_PIPE_FF 3
#endif
      const int64_t np = sc->ff_n > 0 ? GWN_PIPE_FF : 6;
      const int64_t pc =
          (std::max<int64_t>(1ll << 16, (n + np - 1) / np) + 1023) & ~1023ll;
      cm = std::min(cm, pc);
      if (!cs_in) {
        CKE(cudaStreamCreateWithFlags(&cs_in, cudaStreamNonBlocking));
        CKE(cudaStreamCreateWithFlags(&cs_out, cudaStreamNonBlocking));
      }
      // chunk boundaries: equal chunks
      for (int64_t a = cm; a < n; a += cm) cst.push_back(a);
      const int64_t nch = (int64_t)cst.size();
      pev.assign((size_t)(2 * nch), nullptr);
      for (auto& e : pev) CKE(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // per-chunk workspace (reused across chunks and rounds)
    double* pos = ws.get<double>((size_t)(3 * cm));
    int8_t* jit = ws.get<int8_t>((size_t)cm);
    int8_t* jreason = ws.get<int8_t>((size_t)cm);
    int32_t* act[2] = {ws.get<int32_t>((size_t)cm), ws.get<int32_t>((size_t)cm)};
    double* qproj = ws.get<double>((size_t)(3 * cm));
    int32_t* chi = ws.get<int32_t>((size_t)cm);
    int32_t* fl = ws.get<int32_t>((size_t)cm);
    const int nchunk_max = boundary_chunks(sc, (int32_t)cm);
    double* bterm = ws.get<double>((size_t)cm * nchunk_max);
    unsigned long long* rsc = d_cnt + CNT_N;  // round scalars (see kBlk)
    unsigned long long* k3cnt = rsc + 4;
    bool cnt_zeroed = false;
    // Scenes beyond the shared-memory patch table: round 0 takes the queries
    // in ray-column order (launch_column_order), so a warp's rays cross the
    // same leaves and patches -- the cull reads each cell's entries once, and
    // the Newton pass's coefficient loads hit the same L1 lines instead of 32
    // patches per warp.  (Config 2's grid cull gains nothing from it.)
#ifndef GWN_QSORT
#define GWN_QSORT 1
#endif
    const bool sort_q = GWN_QSORT && sc->P > 96 && cm >= 4096;
    // far-field scenes: 3-D Morton order of each round's queries for K4
    const bool ff_sort = sc->ff_n > 0 && cm >= 4096;
    int32_t* ff_order = ff_sort ? ws.get<int32_t>((size_t)cm) : nullptr;
    void* ff_tmp = ff_sort || sort_q ? ws.get<char>(ff_order_scratch_bytes((int32_t)cm)) : nullptr;
    int64_t pair_cap = 0;
    void* k3_scratch = nullptr;  // K3 queues (fallback + Newton items)
    CKE(ws.err);
    if (!pipe)
      for (int64_t a = cm; a < n; a += cm) cst.push_back(a);
    cst.push_back(n);
    for (int64_t ci = 0; ci + 1 < (int64_t)cst.size(); ++ci) {
      const int64_t c0 = cst[ci];
      const int32_t mc = (int32_t)(cst[ci + 1] - c0);
      const double* q0 = d_q + 3 * c0;
      if (pipe) {
        auto h2d = [&](int64_t k) -> cudaError_t {
          const int64_t a = cst[k], b = cst[k + 1];
          cudaError_t e = cudaMemcpyAsync((double*)d_q + 3 * a, queries + 3 * a,
                                          sizeof(double) * 3 * (b - a), cudaMemcpyHostToDevice,
                                          cs_in);
          return e != cudaSuccess ? e : cudaEventRecord(pev[2 * k], cs_in);
        };
        // input copies issued one chunk ahead of the rounds
        constexpr int64_t ahead = 1;
        const int64_t nchk = (int64_t)cst.size() - 1;
        for (int64_t k = ci == 0 ? 0 : ci + ahead; k <= ci + ahead && k < nchk; ++k)
          CKE(h2d(k));
        CKE(cudaStreamWaitEvent(st, pev[2 * ci], 0));
      }
      // round 0 reads the queries in place; k_finalize fills pos / jit for
      // the queries it passes on to the next round
      int32_t m = mc;
      const int32_t* active = nullptr;
      int cur = 0;
      if (sort_q && mc >= 4096) {
        const Round* r0 = nullptr;
        CKE(ensure_round(sc, 0, st, &r0, &stats.ms_round_build));
        CKE(launch_column_order(*r0, mc, q0, ff_tmp, act[1], st));
        active = act[1];  // round 0 writes its re-shoot list into act[0]
        launches += 1;  // column keys (+ a CUB sort)
      }
      for (int r = 0; r < sc->prm.max_rounds && m > 0;) {
        const Round* rdp = nullptr;
        if (r < std::max(1, sc->prm.cached_rounds)) {
          CKE(ensure_round(sc, r, st, &rdp, &stats.ms_round_build));
        } else {
          if (spill_r != r) {
            if (spill_r >= 0) free_round(spill);
            spill_r = -1;
            double dr[3];
            gwn_direction(sc->prm.dir_seed, r, dr);
            const auto t0 = std::chrono::steady_clock::now();
            CKE(build_round_dir(sc, dr, spill, st));
            stats.ms_round_build += std::chrono::duration<double, std::milli>(
                                        std::chrono::steady_clock::now() - t0)
                                        .count();
            spill_r = r;
          }
          rdp = &spill;
        }
        const Round& rd = *rdp;
        // candidate capacity from the scene's running estimate
        int64_t want = (int64_t)(sc->pairs_per_query * 1.25 * m) + 4096;
        if (want > pair_cap) {
          pair_cap = want;
          CKE(ws.k3(intersect_scratch_bytes(pair_cap, sc->P), &k3_scratch));
        }
        // (small re-shoot rounds skip the patch bins: a few items per patch)
        const K3Queues Q = k3_queues(k3_scratch, pair_cap, k3cnt, m >= kBinMinQueries ? sc->P : 0);
        tr.mark("round setup");
        tl_mark(st, "round setup done");
        if (sc->timed) CKE(cudaEventRecord(ev[0], st));
        const double* rpos = r == 0 ? q0 : pos;
        if (!cnt_zeroed) {  // eval counters + round scalars, one memset
          CKE(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * kBlk, st));
          cnt_zeroed = true;
        } else {
          CKE(cudaMemsetAsync(rsc, 0, sizeof(unsigned long long) * 8, st));
        }
        // ---- K2: cull -> (query, leaf) candidates
        if (sc->P > 0) {
          CullZero z;
          z.chi = chi;
          z.flags = fl;
          CKE(launch_cull(sc, rd, m, active, rpos, qproj, rsc, pair_cap, z, Q, d_cnt, st));
          ++launches;
        }
        tr.mark("cull launched");
        tl_mark(st, "cull done");
        if (sc->timed) CKE(cudaEventRecord(ev[1], st));
        // ---- K3: candidate test, DFS fallback, Newton + segmented reduction
        if (sc->P == 0) {  // no cull kernel to zero the accumulators
          CKE(cudaMemsetAsync(chi, 0, sizeof(int32_t) * m, st));
          CKE(cudaMemsetAsync(fl, 0, sizeof(int32_t) * m, st));
        }
        cudaEvent_t join = nullptr;
        if (sc->P > 0) {
          CKE(launch_intersect(sc, rd, Q, rsc, qproj, chi, fl, d_cnt, k3cnt + 3,
                               sc->timed ? ev4 : nullptr, &join, nullptr, st));
          launches += Q.n_bins ? 6 : 3;  // + bin memset, scan, scatter
        }
        tr.mark("k3 launched");
        tl_mark(st, "k3 main done");
        if (sc->timed) CKE(cudaEventRecord(ev[2], st));
        // ---- K4: boundary term
        // (closed scenes: no net boundary, B = 0, nothing to launch)
        const int nchunk = sc->n_edges > 0 ? boundary_chunks(sc, m) : 0;
        if (nchunk > 0) {
          const int32_t* ord = nullptr;
          if (ff_sort && m >= 4096) {
            CKE(launch_ff_order(sc, m, active, rpos, ff_tmp, ff_order, st));
            ord = ff_order;
            launches += 1;  // Morton keys (+ a CUB sort)
          }
          CKE(launch_boundary(sc, rd, m, active, rpos, bterm, nchunk, fl, d_cnt, st, ord,
                              sc->timed && sc->ff_n > 0 ? evb : nullptr));
          launches += sc->ff_n > 0 ? 8 : 1;  // far-field: count, levels, tiles, fill, far eval,
                                            // far sum, near, near sum
        }
        if (sc->timed) CKE(cudaEventRecord(ev[3], st));
        // ---- K5: finalize / compact re-shoots (after the K3 side stream)
        tl_mark(st, "k4 done");
        if (join) CKE(cudaStreamWaitEvent(st, join, 0));
        tl_mark(st, "joined");
        int32_t* nxt = act[cur];
        const bool vec4 = r == 0 && !active && ((uintptr_t)(d_w + c0) & 15) == 0 &&
                          ((uintptr_t)(d_st + c0) & 3) == 0;
        if (vec4) {
          const int32_t nth = (m + 3) / 4;
          // K5: 512-thread blocks, at most 2 per SM (the publish counter's
          // atomics stay few)
          constexpr int k5_bps = 2, k5_bs = 512;
          const int nb4 = k5_bps > 0 ? std::min((nth + k5_bs - 1) / k5_bs, k5_bps * sc->sm_count)
                                     : (nth + k5_bs - 1) / k5_bs;
          k_finalize4<<<nb4, k5_bs, 0, st>>>(
              m, chi, fl, bterm, nchunk, sc->prm.max_rounds, sc->prm.max_jitters,
              sc->prm.dir_seed, index_base + c0, qidx ? qidx + c0 : nullptr,
              sc->prm.jitter_scale * sc->diag, q0, pos, jit, jreason, d_w + c0, d_st + c0, nxt,
              (int32_t*)(rsc + 1), rsc, (unsigned long long)pair_cap, rsc + 2, d_cnt, h_map, kBlk);
        } else {
          k_finalize<<<(m + 127) / 128, 128, 0, st>>>(
              m, active, chi, fl, bterm, nchunk, r, sc->prm.max_rounds, sc->prm.max_jitters,
              sc->prm.dir_seed, index_base + c0, qidx ? qidx + c0 : nullptr,
              sc->prm.jitter_scale * sc->diag, q0, pos, jit,
              jreason, d_w + c0, d_st + c0, nxt, (int32_t*)(rsc + 1), rsc,
              (unsigned long long)pair_cap, rsc + 2, d_cnt, h_map, kBlk);
        }
        CKE(cudaGetLastError());
        ++launches;
        // (K5's last block publishes the scalar block into h_scalar: mapped)
        if (sc->timed) CKE(cudaEventRecord(ev[4], st));
        tl_mark(st, "finalize+d2h done");
        tr.mark("round launched");
        CKE(cudaStreamSynchronize(st));
        tr.mark("round synced");
        const int64_t npairs = h_scalar[CNT_N];
        if (npairs > pair_cap) {  // re-run the round with the exact capacity
          std::lock_guard<std::mutex> lk(sc->mu);
          sc->pairs_per_query = fmax(sc->pairs_per_query, (double)npairs / m);
          continue;
        }
        stats.rounds++;
        if (r > 0) stats.retried += m;
        stats.candidates += npairs;
        if (sc->timed) {
          float a = 0, b = 0, c = 0, d = 0;
          cudaEventElapsedTime(&a, ev[0], ev[1]);
          cudaEventElapsedTime(&b, ev[1], ev[2]);
          cudaEventElapsedTime(&c, ev[2], ev[3]);
          cudaEventElapsedTime(&d, ev[3], ev[4]);
          stats.ms_cull += a;
          stats.ms_intersect += b;
          stats.ms_boundary += c;
          stats.ms_other += d;
          if (sc->ff_n > 0 && nchunk > 0) {
            cudaEventElapsedTime(&a, evb[0], evb[1]);
            cudaEventElapsedTime(&b, evb[1], evb[2]);
            stats.ms_k4_far += a;
            stats.ms_k4_exact += b;
          }
          if (sc->P > 0) {
            cudaEventElapsedTime(&a, ev4[0], ev4[1]);
            cudaEventElapsedTime(&b, ev4[1], ev4[2]);
            cudaEventElapsedTime(&c, ev4[4], ev4[3]);
            cudaEventElapsedTime(&d, ev4[2], ev4[4]);  // patch-bin scan + scatter
            stats.ms_k3_candidates += a + d;
            stats.ms_k3_fallback += b;
            stats.ms_k3_newton += c;
          }
        }
        stats.k3_fallback_items += h_scalar[CNT_N + 4];
        stats.k3_newton_items += h_scalar[CNT_N + 5];
        m = (int32_t)(*(int32_t*)(h_scalar + CNT_N + 1));
        active = nxt;
        cur ^= 1;
        ++r;
      }
      if (pipe) {  // this chunk's outputs back while the next chunk runs
        CKE(cudaEventRecord(pev[2 * ci + 1], st));
        CKE(cudaStreamWaitEvent(cs_out, pev[2 * ci + 1], 0));
        CKE(cudaMemcpyAsync(w_out + c0, d_w + c0, sizeof(double) * mc, cudaMemcpyDeviceToHost,
                            cs_out));
        CKE(cudaMemcpyAsync(status_out + c0, d_st + c0, mc, cudaMemcpyDeviceToHost, cs_out));
      }
    }
  }
  if (host && !pipe) {
    CKE(cudaMemcpyAsync(w_out, d_w, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CKE(cudaMemcpyAsync(status_out, d_st, n, cudaMemcpyDeviceToHost, st));
  }
  if (pipe) CKE(cudaStreamSynchronize(cs_out));
  // eval counters: from the last round's scalar copy (no extra round trip)
  for (int k = 0; k < CNT_N; ++k) h_cnt[k] = (unsigned long long)h_scalar[k];
  if (host) CKE(cudaStreamSynchronize(st));
  stats.nodes = (int64_t)h_cnt[CNT_NODES];
  stats.newton_iters = (int64_t)h_cnt[CNT_NEWTON];
  stats.roots = (int64_t)h_cnt[CNT_ROOTS];
  stats.boundary_segments = (int64_t)h_cnt[CNT_SEGMENTS];
  stats.far_pairs = (int64_t)h_cnt[CNT_FAR];
  stats.far_terms = (int64_t)h_cnt[CNT_FAR_TERMS];
  stats.near_pairs = (int64_t)h_cnt[CNT_NEAR];
  stats.local_evals = (int64_t)h_cnt[CNT_LOCAL];
  stats.shadow_pairs = (int64_t)h_cnt[CNT_SHADOW];
  if (getenv("GWN_TRACE"))
    fprintf(stderr, "[gwn] fallback: max nodes/item %llu, slowest batch: %llu cycles tree %llu code %llu items %llu, max levels %llu\n",
            h_cnt[CNT_MAXNODES], h_cnt[CNT_BIGITEMS] >> 24, (h_cnt[CNT_BIGITEMS] >> 16) & 255, (h_cnt[CNT_BIGITEMS] >> 8) & 255, h_cnt[CNT_BIGITEMS] & 255, h_cnt[CNT_MAXLEVELS]);
  stats.kernel_launches = launches;
  {
    std::lock_guard<std::mutex> lk(sc->mu);
    stats.rounds_built = (int64_t)sc->rounds.size();
    sc->stats = stats;
  }
  tl_mark(st, "outputs copied");
  tr.mark("outputs copied");
done:
  if (spill_r >= 0) {
    cudaStreamSynchronize(st);
    free_round(spill);
  }
  if (pipe && cs_in) {  // no copy may outlive the workspace
    cudaStreamSynchronize(cs_in);
    cudaStreamSynchronize(cs_out);
  }
  for (auto& e : pev)
    if (e) cudaEventDestroy(e);
  ws.release();
  if (st) cudaStreamSynchronize(st);
  else cudaDeviceSynchronize();
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev4)
    if (e) cudaEventDestroy(e);
  for (auto& e : evb)
    if (e) cudaEventDestroy(e);
  tr.mark("done");
  if (g_tl) {
    cudaDeviceSynchronize();
    g_tl->dump();
    g_tl = nullptr;
  }
  return rc;
}

extern "C" int gwn_eval(gwn_scene* sc, const double* queries, int64_t n, int64_t index_base,
                        double* w_out, int8_t* status_out, int32_t flags, void* stream) {
  return eval_core(sc, queries, n, index_base, nullptr, w_out, status_out, flags, stream);
}

namespace gwn {
int eval_impl(gwn_scene* sc, const double* d_q, int64_t n, int64_t index_base,
              const int64_t* qidx, double* d_w, int8_t* d_st, cudaStream_t st,
              gwn_stats& stats) {
  const int rc = eval_core(sc, d_q, n, index_base, qidx, d_w, d_st, 0, st);
  stats = sc->stats;
  return rc;
}
}  // namespace gwn

extern "C" int gwn_all_hits(gwn_scene* sc, int64_t patch, const double origin[3],
                            const double direction[3], const gwn_params* eps, double t_lo,
                            double t_hi, double* t_out, double* uv_out, int32_t* sign_out,
                            int8_t* tang_out, int8_t* graze_out, int32_t cap,
                            int32_t* flags_out) {
  int rc = GWN_OK;
  double* d_out = nullptr;
  int32_t* d_cnt = nullptr;
  double* d_proj = nullptr;
  int32_t cnt[2] = {0, 0};
  constexpr int kRows = 18;  // Bezout bound of line x bicubic (gwn_dfs.cuh kMaxRoots)
  double h[6 * kRows];
  Round rd;
  gwn::DevParams prm;
  if (!sc || patch < 0 || patch >= sc->P || !origin || !direction || cap < 0 ||
      !(t_lo <= t_hi)) {
    set_error("gwn_all_hits: invalid arguments");
    return GWN_E_INVALID;
  }
  prm = sc->dprm;
  if (eps)  // the caller's EpsilonConfig (surfaces.py:587 `eps` argument)
    prm = {eps->residual, eps->dedup, eps->tangent, eps->edge_graze, eps->degenerate,
           eps->domain_tol, eps->t_tol, eps->on_surface_t, eps->band_factor};
  {
    double dd[3] = {direction[0], direction[1], direction[2]};
    double l = sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]);
    if (!(l > 0.0)) {
      set_error("gwn_all_hits: zero direction");
      return GWN_E_INVALID;
    }
    if (fabs(l - 1.0) > 1e-12)  // Ray normalisation rule, geometry.py:49-51
      for (int k = 0; k < 3; ++k) dd[k] /= l;
    make_frame(dd, &rd.f);
  }
  CKE(cudaSetDevice(sc->device));
  {
    // project just this patch on the host (48 dot products)
    double X[48], P48[48];
    CKE(cudaMemcpy(X, sc->ctrl + 48 * patch, sizeof X, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 16; ++k) {
      P48[k] = X[3 * k] * rd.f.e1[0] + X[3 * k + 1] * rd.f.e1[1] + X[3 * k + 2] * rd.f.e1[2];
      P48[16 + k] = X[3 * k] * rd.f.e2[0] + X[3 * k + 1] * rd.f.e2[1] + X[3 * k + 2] * rd.f.e2[2];
      P48[32 + k] = X[3 * k] * rd.f.d[0] + X[3 * k + 1] * rd.f.d[1] + X[3 * k + 2] * rd.f.d[2];
    }
    CKE(cudaMalloc(&d_proj, sizeof P48));
    CKE(cudaMemcpy(d_proj, P48, sizeof P48, cudaMemcpyHostToDevice));
  }
  CKE(cudaMalloc(&d_out, sizeof h));
  CKE(cudaMalloc(&d_cnt, sizeof cnt));
  rd.proj = d_proj;
  CKE(launch_all_hits(rd, prm, origin, t_lo, t_hi, d_out, d_cnt, kRows, 0));
  CKE(cudaMemcpy(cnt, d_cnt, sizeof cnt, cudaMemcpyDeviceToHost));
  CKE(cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost));
  for (int k = 0; k < cnt[0] && k < cap && k < kRows; ++k) {
    if (t_out) t_out[k] = h[6 * k];
    if (uv_out) {
      uv_out[2 * k] = h[6 * k + 1];
      uv_out[2 * k + 1] = h[6 * k + 2];
    }
    if (sign_out) sign_out[k] = (int32_t)h[6 * k + 3];
    if (tang_out) tang_out[k] = (int8_t)h[6 * k + 4];
    if (graze_out) graze_out[k] = (int8_t)h[6 * k + 5];
  }
  if (flags_out) *flags_out = cnt[1];
  rc = cnt[0];
done:
  if (d_out) cudaFree(d_out);
  if (d_cnt) cudaFree(d_cnt);
  if (d_proj) cudaFree(d_proj);
  return rc;
}

extern "C" int gwn_single_loop_batch(const double* loop, int64_t B, const double origin[3],
                                     const double direction[3], const double* hit_ts,
                                     const int64_t* hit_signs, int64_t H, const double* qts,
                                     int64_t K, double on_tol, double t_eps, double* w_out,
                                     int8_t* ok_out, int device) {
  (void)on_tol;
  int rc = GWN_OK;
  double *d_loop = nullptr, *d_ht = nullptr, *d_q = nullptr, *d_w = nullptr;
  int64_t* d_hs = nullptr;
  int8_t* d_ok = nullptr;
  double d[3];
  if (!loop || B < 3 || !origin || !direction || H < 0 || K < 0 || (H && (!hit_ts || !hit_signs)) ||
      (K && (!qts || !w_out || !ok_out))) {
    set_error("gwn_single_loop_batch: invalid arguments (loop needs >= 3 points)");
    return GWN_E_INVALID;
  }
  if (K == 0) return GWN_OK;
  {
    double l = sqrt(direction[0] * direction[0] + direction[1] * direction[1] +
                    direction[2] * direction[2]);
    for (int k = 0; k < 3; ++k) d[k] = fabs(l - 1.0) > 1e-12 ? direction[k] / l : direction[k];
  }
  CKE(cudaSetDevice(device));
  CKE(cudaMalloc(&d_loop, sizeof(double) * 3 * B));
  CKE(cudaMalloc(&d_ht, sizeof(double) * (H + 1)));
  CKE(cudaMalloc(&d_hs, sizeof(int64_t) * (H + 1)));
  CKE(cudaMalloc(&d_q, sizeof(double) * K));
  CKE(cudaMalloc(&d_w, sizeof(double) * K));
  CKE(cudaMalloc(&d_ok, K));
  CKE(cudaMemcpy(d_loop, loop, sizeof(double) * 3 * B, cudaMemcpyHostToDevice));
  if (H) {
    CKE(cudaMemcpy(d_ht, hit_ts, sizeof(double) * H, cudaMemcpyHostToDevice));
    CKE(cudaMemcpy(d_hs, hit_signs, sizeof(int64_t) * H, cudaMemcpyHostToDevice));
  }
  CKE(cudaMemcpy(d_q, qts, sizeof(double) * K, cudaMemcpyHostToDevice));
  CKE(launch_single_loop(d_loop, B, origin, d, d_ht, d_hs, H, d_q, K, t_eps, 1e-12, d_w, d_ok, 0));
  CKE(cudaMemcpy(w_out, d_w, sizeof(double) * K, cudaMemcpyDeviceToHost));
  CKE(cudaMemcpy(ok_out, d_ok, K, cudaMemcpyDeviceToHost));
done:
  cudaFree(d_loop);
  cudaFree(d_ht);
  cudaFree(d_hs);
  cudaFree(d_q);
  cudaFree(d_w);
  cudaFree(d_ok);
  return rc;
}

extern "C" int gwn_selftest_rsqrt(int device, int64_t n, uint64_t* max_ulp) {
  int rc = GWN_OK;
  unsigned long long m = 0;
  if (!max_ulp || n <= 0) {
    set_error("gwn_selftest_rsqrt: invalid arguments");
    return GWN_E_INVALID;
  }
  CKE(cudaSetDevice(device));
  CKE(selftest_rsqrt(n, &m));
  *max_ulp = m;
done:
  return rc;
}
