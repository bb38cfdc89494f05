// gwn_rays.cu -- ray reuse: winding numbers of many
// points along a batch of parallel rays with ONE intersection pass per ray.
//
// Reference: SPEC.md:381-389 `winding_numbers_along_ray` ("one all-hits
// intersection per ray; chi from cached hits with t_j > t")
// slice / voxelize ("min(W,H) rays", "N^2 rays"), and the
// reference's batch kernel `single_loop_batch` (_kernels.py:801-823, cached
// hit_ts / hit_signs, clash test :782-784).
//
// B200 path: the rays of a batch share one direction, so they form a round
// of their own (projection, leaves, cull grid for that direction, cached per
// scene).  K2 + K3 run once per RAY in record mode, appending every owned
// root (ray, t, sign).  Per point: chi = sum of the signs of its ray's hits
// beyond it (a hit within on_surface_t of the point is a clash), the K4
// boundary term in the ray direction, w = chi + B.  Points whose ray had a
// tangent / grazing hit, or that clash, are degenerate or hit the band, are
// re-evaluated through the per-point engine (re-shoot and jitter policy).
#include <cub/cub.cuh>

#include <math.h>
#include <string.h>

#include "gwn_internal.h"
#include "gwn_k3.cuh"

namespace gwn {

// start point of each ray: a margin before its first parameter
__global__ void k_ray_starts(int64_t R, const double* __restrict__ org,
                             const double* __restrict__ ts, const int64_t* __restrict__ offs,
                             Frame f, double margin, double* __restrict__ rpos,
                             double* __restrict__ rt0) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t a = offs[r], b = offs[r + 1];
  const double t0 = (b > a ? ts[a] : 0.0) - margin;
  rt0[r] = t0;
  for (int k = 0; k < 3; ++k) rpos[3 * r + k] = org[3 * r + k] + t0 * f.d[k];
}

__global__ void k_hit_hist(const HitRec* __restrict__ rec, int64_t n, unsigned long long* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[rec[i].slot], 1ull);
}

__global__ void k_hit_scatter(const HitRec* __restrict__ rec, int64_t n,
                              const int64_t* __restrict__ hoff, unsigned long long* __restrict__ cursor,
                              const double* __restrict__ rt0, double* __restrict__ ht,
                              int32_t* __restrict__ hs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const HitRec h = rec[i];
  const int64_t k = hoff[h.slot] + (int64_t)atomicAdd(&cursor[h.slot], 1ull);
  ht[k] = rt0[h.slot] + h.t;  // absolute ray parameter
  hs[k] = h.sign;
}

// per point (global index g in [p0, p0+np)): position, chi from its ray's hits
__global__ void k_ray_points(int64_t p0, int64_t np, int64_t R, const double* __restrict__ org,
                             const double* __restrict__ ts, const int64_t* __restrict__ offs,
                             Frame f, const int64_t* __restrict__ hoff,
                             const double* __restrict__ ht, const int32_t* __restrict__ hs,
                             const int32_t* __restrict__ rflags, double on_surface_t,
                             double* __restrict__ pos, int32_t* __restrict__ chi,
                             int32_t* __restrict__ qfl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  const int64_t g = p0 + i;
  // ray of point g: last r with offs[r] <= g
  int64_t lo = 0, hi = R - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (offs[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  const int64_t r = lo;
  const double t = ts[g];
  for (int k = 0; k < 3; ++k) pos[3 * i + k] = org[3 * r + k] + t * f.d[k];
  int32_t c = 0, fl = rflags[r] & FLAG_RESHOOT;
  for (int64_t h = hoff[r]; h < hoff[r + 1]; ++h) {
    const double th = ht[h];
    if (fabs(th - t) <= on_surface_t) fl |= FLAG_ONSURF;  // clash (_kernels.py:782-784)
    if (th > t) c += hs[h];
  }
  chi[i] = c;
  qfl[i] = fl;
}

__global__ void k_ray_finalize(int64_t np, const int32_t* __restrict__ chi,
                               const int32_t* __restrict__ qfl, const double* __restrict__ bpart,
                               int nchunk, double* __restrict__ w, int8_t* __restrict__ stt,
                               int64_t* __restrict__ fb, unsigned long long* __restrict__ nfb,
                               int64_t p0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  double ang = 0.0;
  for (int c = 0; c < nchunk; ++c) ang = __dadd_rn(ang, bpart[(int64_t)c * np + i]);
  w[i] = __dadd_rn((double)chi[i], __dmul_rn(ang, 0.15915494309189533576888));
  stt[i] = GWN_STATUS_OK;
  if (qfl[i]) {  // per-point engine (new direction / jitter)
    const unsigned long long k = atomicAdd(nfb, 1ull);
    fb[k] = p0 + i;
  }
}

__global__ void k_gather_pos(int64_t n, const int64_t* __restrict__ idx,
                             const double* __restrict__ org, const double* __restrict__ ts,
                             const int64_t* __restrict__ offs, int64_t R, Frame f,
                             double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t g = idx[i];
  int64_t lo = 0, hi = R - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (offs[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  for (int k = 0; k < 3; ++k) out[3 * i + k] = org[3 * lo + k] + ts[g] * f.d[k];
}

__global__ void k_scatter_fb(int64_t n, const int64_t* __restrict__ idx,
                             const double* __restrict__ fw, const int8_t* __restrict__ fs,
                             double* __restrict__ w, int8_t* __restrict__ stt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  w[idx[i]] = fw[i];
  stt[idx[i]] = fs[i];
}

}  // namespace gwn

using namespace gwn;

#define CKR(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      set_error("%s failed: %s", #call, cudaGetErrorString(e_));              \
      rc = (e_ == cudaErrorMemoryAllocation) ? GWN_E_OOM : GWN_E_CUDA;         \
      goto done;                                                               \
    }                                                                          \
  } while (0)

// Round for an explicit ray direction: cached per scene (up to kDirCache
// directions, never evicted, so a cached Round* stays valid for the scene's
// lifetime); past the cache the call builds a private round (*owned) that it
// frees when done.
constexpr size_t kDirCache = 8;
static cudaError_t dir_round(gwn_scene* sc, const double d[3], Round** out, Round* owned,
                             bool* is_owned, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(sc->mu);
  *is_owned = false;
  for (auto& kv : sc->dir_rounds)
    if (kv.first[0] == d[0] && kv.first[1] == d[1] && kv.first[2] == d[2]) {
      *out = &kv.second;
      return cudaSuccess;
    }
  Round rd;
  cudaError_t e = build_round_dir(sc, d, rd, st);
  if (e != cudaSuccess) return e;
  if (sc->dir_rounds.size() >= kDirCache) {
    *owned = rd;
    *is_owned = true;
    *out = owned;
    return cudaSuccess;
  }
  sc->dir_rounds.push_back({{d[0], d[1], d[2]}, rd});
  *out = &sc->dir_rounds.back().second;
  return cudaSuccess;
}

template <class T>
static T* dalloc(std::vector<void*>& v, size_t n, cudaStream_t st, cudaError_t& e) {
  void* p = nullptr;
  if (e != cudaSuccess) return nullptr;
  e = cudaMallocAsync(&p, n * sizeof(T) + 16, st);
  if (e == cudaSuccess) v.push_back(p);
  return (T*)p;
}

extern "C" int gwn_eval_rays(gwn_scene* sc, const double* origins, int64_t R,
                             const double direction[3], const double* ts, const int64_t* offs,
                             double* w_out, int8_t* status_out, int32_t flags, void* stream,
                             int64_t* rays_cast) {
  int rc = GWN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<void*> bufs;
  cudaError_t ae = cudaSuccess;
  const bool host = (flags & GWN_HOST_BUFFERS) != 0;
  int64_t nq = 0;
  double d[3];
  Round* rd = nullptr;
  Round rd_owned;
  bool rd_is_owned = false;
  gwn_stats stats;
  memset(&stats, 0, sizeof stats);
  if (!sc || R < 0 || !direction || (R > 0 && (!origins || !ts || !offs || !w_out || !status_out))) {
    set_error("gwn_eval_rays: invalid arguments");
    return GWN_E_INVALID;
  }
  if (rays_cast) *rays_cast = 0;
  if (R == 0) return GWN_OK;
  {
    const double l = sqrt(direction[0] * direction[0] + direction[1] * direction[1] +
                          direction[2] * direction[2]);
    if (!(l > 0.0)) {
      set_error("gwn_eval_rays: zero direction");
      return GWN_E_INVALID;
    }
    for (int k = 0; k < 3; ++k) d[k] = direction[k] / l;
  }
  CKR(cudaSetDevice(sc->device));
  {
    // inputs on the device
    const double* d_org = origins;
    const double* d_ts = ts;
    const int64_t* d_offs = offs;
    double* d_w = w_out;
    int8_t* d_st = status_out;
    if (host) {
      nq = offs[R];
      double* o = dalloc<double>(bufs, 3 * R, st, ae);
      double* t = dalloc<double>(bufs, nq + 1, st, ae);
      int64_t* f = dalloc<int64_t>(bufs, R + 1, st, ae);
      d_w = dalloc<double>(bufs, nq + 1, st, ae);
      d_st = dalloc<int8_t>(bufs, nq + 1, st, ae);
      CKR(ae);
      CKR(cudaMemcpyAsync(o, origins, sizeof(double) * 3 * R, cudaMemcpyHostToDevice, st));
      CKR(cudaMemcpyAsync(t, ts, sizeof(double) * nq, cudaMemcpyHostToDevice, st));
      CKR(cudaMemcpyAsync(f, offs, sizeof(int64_t) * (R + 1), cudaMemcpyHostToDevice, st));
      d_org = o;
      d_ts = t;
      d_offs = f;
    } else {
      CKR(cudaMemcpyAsync(&nq, offs + R, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CKR(cudaStreamSynchronize(st));
    }
    if (nq > 0) {
      CKR(dir_round(sc, d, &rd, &rd_owned, &rd_is_owned, st));
      const int32_t m = (int32_t)R;
      double* rpos = dalloc<double>(bufs, 3 * R, st, ae);
      double* rt0 = dalloc<double>(bufs, R, st, ae);
      double* qproj = dalloc<double>(bufs, 3 * R, st, ae);
      int32_t* rchi = dalloc<int32_t>(bufs, R, st, ae);
      int32_t* rfl = dalloc<int32_t>(bufs, R, st, ae);
      unsigned long long* cnt = dalloc<unsigned long long>(bufs, CNT_N + 12, st, ae);
      CKR(ae);
      unsigned long long* rsc = cnt + CNT_N;  // [0] candidates, [4] records, [8..11] K3 counters
      CKR(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (CNT_N + 12), st));
      k_ray_starts<<<(unsigned)((R + 127) / 128), 128, 0, st>>>(
          R, d_org, d_ts, d_offs, rd->f, 1e-6 * (1.0 + sc->diag), rpos, rt0);
      CKR(cudaGetLastError());
      // ---- K2 + K3 once per ray, record mode (re-run on buffer overflow)
      int64_t pair_cap = (int64_t)(sc->pairs_per_query * 1.25 * R) + 4096;
      int64_t nrec = 0;
      HitRec* rec = nullptr;
      for (;;) {
        std::vector<void*> rb;
        void* scratch = dalloc<char>(rb, intersect_scratch_bytes(pair_cap, sc->P), st, ae);
        const int64_t rcap = 2 * pair_cap + 1024;
        rec = dalloc<HitRec>(bufs, rcap, st, ae);
        CKR(ae);
        CKR(cudaMemsetAsync(rsc, 0, sizeof(unsigned long long) * 12, st));
        const K3Queues Q = k3_queues(scratch, pair_cap, rsc + 8, m >= kBinMinQueries ? sc->P : 0);
        CullZero z;
        z.chi = rchi;
        z.flags = rfl;
        CKR(launch_cull(sc, *rd, m, nullptr, rpos, qproj, rsc, pair_cap, z, Q, cnt, st));
        RecordSink sink{rec, rsc + 4, (unsigned long long)rcap};
        cudaEvent_t join = nullptr;
        CKR(launch_intersect(sc, *rd, Q, rsc, qproj, rchi, rfl, cnt, rsc + 11, nullptr, &join,
                             &sink, st));
        if (join) CKR(cudaStreamWaitEvent(st, join, 0));
        unsigned long long h[8];
        CKR(cudaMemcpyAsync(h, rsc, sizeof h, cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        for (void* p : rb) cudaFreeAsync(p, st);
        stats.candidates += (int64_t)h[0];
        if ((int64_t)h[0] > pair_cap) {
          std::lock_guard<std::mutex> lk(sc->mu);
          sc->pairs_per_query = fmax(sc->pairs_per_query, (double)h[0] / R);
          pair_cap = (int64_t)(h[0] * 1.25) + 4096;
          continue;
        }
        nrec = (int64_t)(h[4] < (unsigned long long)rcap ? h[4] : rcap);
        break;
      }
      // ---- group the hits by ray (counting sort)
      unsigned long long* hcnt = dalloc<unsigned long long>(bufs, R + 1, st, ae);
      unsigned long long* hoffu = dalloc<unsigned long long>(bufs, R + 1, st, ae);
            double* ht = dalloc<double>(bufs, nrec + 1, st, ae);
      int32_t* hs = dalloc<int32_t>(bufs, nrec + 1, st, ae);
      CKR(ae);
      CKR(cudaMemsetAsync(hcnt, 0, sizeof(unsigned long long) * (R + 1), st));
      if (nrec > 0)
        k_hit_hist<<<(unsigned)((nrec + 255) / 256), 256, 0, st>>>(rec, nrec, hcnt);
      {
        size_t tb = 0;
        CKR(cub::DeviceScan::ExclusiveSum(nullptr, tb, hcnt, hoffu, (int)(R + 1), st));
        void* tmp = dalloc<char>(bufs, tb, st, ae);
        CKR(ae);
        CKR(cub::DeviceScan::ExclusiveSum(tmp, tb, hcnt, hoffu, (int)(R + 1), st));
      }
      const int64_t* hoff = (const int64_t*)hoffu;
      CKR(cudaMemsetAsync(hcnt, 0, sizeof(unsigned long long) * (R + 1), st));
      if (nrec > 0)
        k_hit_scatter<<<(unsigned)((nrec + 255) / 256), 256, 0, st>>>(rec, nrec, hoff, hcnt, rt0,
                                                                      ht, hs);
      CKR(cudaGetLastError());
            // ---- per point: chi, K4, w (in chunks of points)
      const int64_t chunk = 1ll << 21;
      const int64_t cm = nq < chunk ? nq : chunk;
      const int nch = boundary_chunks(sc, (int32_t)cm);
      double* pos = dalloc<double>(bufs, 3 * cm, st, ae);
      int32_t* chi = dalloc<int32_t>(bufs, cm, st, ae);
      int32_t* qfl = dalloc<int32_t>(bufs, cm, st, ae);
      double* bpart = dalloc<double>(bufs, (size_t)cm * nch, st, ae);
      int64_t* fb = dalloc<int64_t>(bufs, nq + 1, st, ae);
      unsigned long long* nfb = dalloc<unsigned long long>(bufs, 1, st, ae);
      CKR(ae);
      CKR(cudaMemsetAsync(nfb, 0, sizeof(unsigned long long), st));
      for (int64_t p0 = 0; p0 < nq; p0 += cm) {
        const int64_t np = (nq - p0) < cm ? (nq - p0) : cm;
        const unsigned g = (unsigned)((np + 127) / 128);
        k_ray_points<<<g, 128, 0, st>>>(p0, np, R, d_org, d_ts, d_offs, rd->f, hoff, ht, hs, rfl,
                                        sc->dprm.on_surface_t, pos, chi, qfl);
        CKR(cudaGetLastError());
        if (sc->n_edges > 0)
          CKR(launch_boundary(sc, *rd, (int32_t)np, nullptr, pos, bpart, nch, qfl, cnt, st));
        k_ray_finalize<<<g, 128, 0, st>>>(np, chi, qfl, bpart, sc->n_edges > 0 ? nch : 0,
                                          d_w + p0, d_st + p0, fb, nfb, p0);
        CKR(cudaGetLastError());
      }
      // ---- points that need the per-point engine (re-shoot / jitter)
      unsigned long long hnfb = 0;
      CKR(cudaMemcpyAsync(&hnfb, nfb, sizeof hnfb, cudaMemcpyDeviceToHost, st));
      CKR(cudaStreamSynchronize(st));
      if (hnfb > 0) {
        const int64_t nf = (int64_t)hnfb;
        double* fpos = dalloc<double>(bufs, 3 * nf, st, ae);
        double* fw = dalloc<double>(bufs, nf, st, ae);
        int8_t* fs = dalloc<int8_t>(bufs, nf, st, ae);
        CKR(ae);
        k_gather_pos<<<(unsigned)((nf + 127) / 128), 128, 0, st>>>(nf, fb, d_org, d_ts, d_offs, R,
                                                                   rd->f, fpos);
        CKR(cudaGetLastError());
        gwn_stats fst;
        rc = eval_impl(sc, fpos, nf, 0, fb, fw, fs, st, fst);
        if (rc < 0) goto done;
        k_scatter_fb<<<(unsigned)((nf + 127) / 128), 128, 0, st>>>(nf, fb, fw, fs, d_w, d_st);
        CKR(cudaGetLastError());
        stats.retried = nf;
      }
      if (host) {
        CKR(cudaMemcpyAsync(w_out, d_w, sizeof(double) * nq, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(status_out, d_st, nq, cudaMemcpyDeviceToHost, st));
      }
      unsigned long long hc[CNT_N];
      CKR(cudaMemcpyAsync(hc, cnt, sizeof hc, cudaMemcpyDeviceToHost, st));
      CKR(cudaStreamSynchronize(st));
      stats.queries = nq;
      stats.rounds = 1;
      stats.nodes = (int64_t)hc[CNT_NODES];
      stats.newton_iters = (int64_t)hc[CNT_NEWTON];
      stats.roots = (int64_t)hc[CNT_ROOTS];
      stats.boundary_segments = (int64_t)hc[CNT_SEGMENTS];
      stats.far_pairs = (int64_t)hc[CNT_FAR];
      {
    std::lock_guard<std::mutex> lk(sc->mu);
    sc->stats = stats;
  }
      if (rays_cast) *rays_cast = R;
    }
  }
done:
  for (void* p : bufs) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  if (rd_is_owned) free_round(rd_owned);
  return rc;
}
