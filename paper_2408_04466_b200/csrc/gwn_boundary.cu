// gwn_boundary.cu -- K4: per-query boundary term over the net boundary.
//
// The reference evaluates the boundary correction per query by projecting
// the loop to the unit sphere, testing it for self-crossings, summing
// Gauss-Bonnet turning angles and locating the ray direction relative to the
// loop (_kernels.py:723-798); the generic case needs the SPEC arrangement
// (SPEC.md:240-336).  Both equal the arrangement-free fan sum
//     B(p, d) = (1/4pi) sum_e 2 atan2(c.(a^ x b^), 1 + a^.b^ + b^.c + c.a^),
// c = -d, over the loop segments (a, b) (pinned against the
// fixed single_loop_batch to 2.3e-13 by tests/test_oracle_golden.py).
//
// B200 formulation.  With unit vectors a^, b^ and d = -c the van Oosterom
// terms are rewritten exactly in the shifted variables u = a^ - d, v = b^ - d:
//     1 + a^.b^ + b^.c + c.a^ = u.v,     c.(a^ x b^) = -(d x u).v
// which keeps full relative accuracy when d points at a segment (u, v small;
// the plain form cancels catastrophically there -- measured 7e-9 drift on
// config 5).  The per-segment atan2 is replaced by a running complex product
// Z *= (u.v + i num) with an exact branch-cut counter from sign bits and a
// power-of-two renormalisation every 8 segments; one atan2 per query.
// Per vertex: 3 DADD, |r|^2, rsqrt, 3 DFMA for u, d x u; per segment: 2 dot
// products + 4 for the complex product.  Boundary vertices (x,y,z) are
// staged in shared-memory tiles and read as warp-wide broadcasts.
#include <algorithm>

#include "gwn_internal.h"

namespace gwn {

constexpr int kTileV = 2000;   // vertices per shared-memory tile (3 x 2000 x 8 B = 48 KB)
constexpr int kBlockQ = 256;   // queries (threads) per block

struct SegState {
  double Zr, Zi;
  int wraps;
};

__device__ __forceinline__ bool signbit_hi(double x) { return __double2hiint(x) < 0; }

// multiply Z by (den + i num) with exact branch-cut bookkeeping
__device__ __forceinline__ void cmul_track(SegState& s, double den, double num) {
  double zr = s.Zr * den - s.Zi * num;
  double zi = s.Zr * num + s.Zi * den;
  bool a = signbit_hi(s.Zi), b = signbit_hi(num), c = signbit_hi(zi);
  s.wraps += (!a && !b && c) ? 1 : 0;
  s.wraps -= (a && b && !c) ? 1 : 0;
  s.Zr = zr;
  s.Zi = zi;
}

__device__ __forceinline__ void renorm(SegState& s) {
  double m = fmax(fabs(s.Zr), fabs(s.Zi));
  int e = ((__double2hiint(m) >> 20) & 0x7ff);
  if (e == 0 || e == 0x7ff) return;  // zero/denormal/non-finite: degenerate, flagged elsewhere
  double sc = __hiloint2double((2046 - e) << 20, 0);  // 2^(1023-e), exact
  s.Zr *= sc;
  s.Zi *= sc;
}

// Per-vertex quantities of the shifted fan formula.
struct Vtx {
  double ux, uy, uz;   // a^ - d
  double gx, gy, gz;   // d x u
  double l;            // |x - p|
  bool ok;
};

__device__ __forceinline__ Vtx make_vtx(double x, double y, double z, double px, double py,
                                        double pz, double dx, double dy, double dz, double deg) {
  Vtx v;
  const double rx = x - px, ry = y - py, rz = z - pz;
  const double l2 = rx * rx + ry * ry + rz * rz;
  const double il = rsqrt(l2);
  v.l = l2 * il;
  v.ok = v.l >= deg;
  v.ux = fma(rx, il, -dx);
  v.uy = fma(ry, il, -dy);
  v.uz = fma(rz, il, -dz);
  v.gx = dy * v.uz - dz * v.uy;
  v.gy = dz * v.ux - dx * v.uz;
  v.gz = dx * v.uy - dy * v.ux;
  return v;
}

// polyline/curve band test (rare path, den < 0): d within band_factor*h/dist
// of the arc (a, b).  Raw offsets are recovered as (u + d) * l.
__device__ __forceinline__ bool band_hit(const Vtx& a, const Vtx& b, double num, double dx,
                                      double dy, double dz, double h, double band_factor) {
  const double ax = a.ux + dx, ay = a.uy + dy, az = a.uz + dz;
  const double bx = b.ux + dx, by = b.uy + dy, bz = b.uz + dz;
  const double sgx = bx * b.l - ax * a.l, sgy = by * b.l - ay * a.l, sgz = bz * b.l - az * a.l;
  const double L = sqrt(sgx * sgx + sgy * sgy + sgz * sgz);
  const double dist = fmin(a.l, b.l) - L;
  if (dist <= 0.0) return true;
  const double cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
  const double s2 = cx * cx + cy * cy + cz * cz;
  const double th = band_factor * h / dist;
  return num * num <= th * th * s2;
}

// One segment (a, b): accumulate; the band test runs only when den < 0.
__device__ __forceinline__ void fan_segment(SegState& st, const Vtx& a, const Vtx& b, double dx,
                                            double dy, double dz, const double* band_h,
                                            int64_t e, double band_factor, int& flags) {
  const double den = a.ux * b.ux + a.uy * b.uy + a.uz * b.uz;
  const double num = -(a.gx * b.ux + a.gy * b.uy + a.gz * b.uz);
  const bool ok = a.ok && b.ok;
  if (den < 0.0 && ok && band_h) {
    if (band_hit(a, b, num, dx, dy, dz, __ldg(band_h + e), band_factor)) flags |= FLAG_BAND;
  }
  cmul_track(st, ok ? den : 1.0, ok ? num : 0.0);
}

template <int QPT>
__global__ void __launch_bounds__(kBlockQ)
k_boundary(int32_t m, const int32_t* __restrict__ active, const double* __restrict__ pos,
           const double* __restrict__ verts, int64_t V, int S, int64_t n_edges,
           const double* __restrict__ band_h, Frame f, DevParams prm,
           double* __restrict__ bpart, int32_t* __restrict__ flag_acc,
           unsigned long long* __restrict__ counters) {
  // blockIdx.y: chunk of whole edges [e0, e1) -> vertex range [v0, v1)
  const int nchunk = gridDim.y;
  const int64_t e0 = n_edges * blockIdx.y / nchunk, e1 = n_edges * (blockIdx.y + 1) / nchunk;
  const int64_t vbeg = e0 * S, vend = e1 * S;
  __shared__ double sx[kTileV], sy[kTileV], sz[kTileV];
  const double dx = f.d[0], dy = f.d[1], dz = f.d[2];
  const double deg = prm.degenerate;
  int32_t slot[QPT];
  double px[QPT], py[QPT], pz[QPT];
  SegState st[QPT];
  int flags[QPT];
  Vtx va[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    slot[j] = blockIdx.x * (blockDim.x * QPT) + j * blockDim.x + threadIdx.x;
    const bool live = slot[j] < m;
    const int32_t q = live ? (active ? active[slot[j]] : slot[j]) : 0;
    px[j] = live ? pos[3 * (int64_t)q] : 0.0;
    py[j] = live ? pos[3 * (int64_t)q + 1] : 0.0;
    pz[j] = live ? pos[3 * (int64_t)q + 2] : 0.0;
    st[j] = SegState{1.0, 0.0, 0};
    flags[j] = 0;
    va[j].ok = false;
  }
  int nseg = 0;
  for (int64_t t0 = vbeg; t0 < vend; t0 += kTileV) {
    const int nt = (int)min((int64_t)kTileV, vend - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
      const int64_t g = t0 + k;
      sx[k] = verts[g];
      sy[k] = verts[V + g];
      sz[k] = verts[2 * V + g];
    }
    __syncthreads();
    int64_t e = t0 / S;               // edge of the tile's first vertex
    int kin = (int)(t0 - e * S);      // its index within that edge
    for (int k = 0; k < nt; ++k) {
      const double x = sx[k], y = sy[k], z = sz[k];
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        const Vtx vb = make_vtx(x, y, z, px[j], py[j], pz[j], dx, dy, dz, deg);
        if (!vb.ok) flags[j] |= FLAG_DEGEN;
        if (kin != 0) fan_segment(st[j], va[j], vb, dx, dy, dz, band_h, e, prm.band_factor, flags[j]);
        va[j] = vb;
      }
      if (kin != 0 && (++nseg & 7) == 0) {
#pragma unroll
        for (int j = 0; j < QPT; ++j) renorm(st[j]);
      }
      if (++kin == S) {
        kin = 0;
        ++e;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    if (slot[j] < m) {
      // partial angle sum of this edge chunk; K5 adds the chunks in order
      bpart[(int64_t)blockIdx.y * m + slot[j]] =
          atan2(st[j].Zi, st[j].Zr) + 6.283185307179586476925 * (double)st[j].wraps;
      if (flags[j]) atomicOr(&flag_acc[slot[j]], flags[j]);
    }
  }
  if (threadIdx.x == 0) {
    int32_t nq = min((int32_t)(blockDim.x * QPT), m - (int32_t)(blockIdx.x * blockDim.x * QPT));
    int64_t segs = (vend - vbeg) - (e1 - e0);
    atomicAdd(&counters[CNT_SEGMENTS], (unsigned long long)(segs * nq));
  }
}

constexpr int kQPT = 2;

// Edge chunks of the boundary sum.  Fixed per scene (not per batch) so the
// chunk partials -- added in chunk order by K5 -- make w bit-identical for any
// batching, chunking or sharding of the queries; enough chunks that small
// batches still fill the GPU.
int boundary_chunks(const gwn_scene* sc, int32_t m) {
  (void)m;
  if (sc->n_edges <= 0) return 1;
  return (int)std::min<int64_t>(sc->n_edges, 64);
}

cudaError_t launch_boundary(const gwn_scene* sc, const Round& rd, int32_t m,
                            const int32_t* active, const double* pos, double* bpart, int nchunk,
                            int32_t* flags, unsigned long long* counters, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  int64_t V = sc->n_edges * sc->S;
  if (V == 0) return cudaMemsetAsync(bpart, 0, sizeof(double) * m, st);
  dim3 grid((m + kBlockQ * kQPT - 1) / (kBlockQ * kQPT), nchunk);
  k_boundary<kQPT><<<grid, kBlockQ, 0, st>>>(m, active, pos, sc->verts, V, sc->S, sc->n_edges,
                                             sc->band_h, rd.f, sc->dprm, bpart, flags, counters);
  return cudaGetLastError();
}

// _kernels.single_loop_batch (_kernels.py:801-823) on the GPU: one closed loop,
// queries p_k = o + t_k d on one ray, chi from the cached hits with t_h > t_k
// (:778-788).  ok = 0 only for a hit clash |t_h - t_k| <= t_eps or a
// degenerate projection; the fan formula needs no simple-loop restriction.
__global__ void k_single_loop(const double* __restrict__ loop, int64_t B, double ox, double oy,
                              double oz, double dx, double dy, double dz,
                              const double* __restrict__ hit_ts,
                              const int64_t* __restrict__ hit_signs, int64_t H,
                              const double* __restrict__ qts, int64_t K, double t_eps,
                              double deg, double* __restrict__ w, int8_t* __restrict__ ok) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double t = qts[k];
  const double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
  long long chi = 0;
  bool clash = false;
  for (int64_t h = 0; h < H; ++h) {
    if (fabs(hit_ts[h] - t) <= t_eps) clash = true;
    if (hit_ts[h] > t) chi += hit_signs[h];
  }
  SegState st = {1.0, 0.0, 0};
  bool bad = false;
  Vtx va = make_vtx(loop[3 * (B - 1)], loop[3 * (B - 1) + 1], loop[3 * (B - 1) + 2], px, py, pz,
                    dx, dy, dz, deg);
  int flags = 0;
  for (int64_t i = 0; i < B; ++i) {
    Vtx vb = make_vtx(loop[3 * i], loop[3 * i + 1], loop[3 * i + 2], px, py, pz, dx, dy, dz, deg);
    if (!va.ok || !vb.ok) bad = true;
    fan_segment(st, va, vb, dx, dy, dz, nullptr, 0, 0.0, flags);
    if ((i & 7) == 7) renorm(st);
    va = vb;
  }
  const double ang = atan2(st.Zi, st.Zr) + 6.283185307179586476925 * (double)st.wraps;
  w[k] = (double)chi + ang * 0.15915494309189533576888;
  ok[k] = (clash || bad) ? 0 : 1;
}

cudaError_t launch_single_loop(const double* loop, int64_t B, const double* o, const double* d,
                               const double* hit_ts, const int64_t* hit_signs, int64_t H,
                               const double* qts, int64_t K, double t_eps, double deg, double* w,
                               int8_t* ok, cudaStream_t st) {
  if (K <= 0) return cudaSuccess;
  k_single_loop<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(loop, B, o[0], o[1], o[2], d[0],
                                                             d[1], d[2], hit_ts, hit_signs, H,
                                                             qts, K, t_eps, deg, w, ok);
  return cudaGetLastError();
}

}  // namespace gwn
