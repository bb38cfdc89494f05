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
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "gwn_fan.cuh"
#include "gwn_farfield.cuh"

namespace gwn {

constexpr int kTileV = 2000;   // vertices per shared-memory tile (3 x 2000 x 8 B = 48 KB)
constexpr int kBlockQ = 256;   // queries (threads) per block

// Per-vertex quantities of the shifted fan formula in the round's ray frame
// (e1, e2, d): d = (0,0,1), so u = r/|r| - d = (rx il, ry il, rz il - 1).
struct VtxF {
  double ux, uy, uz;   // a^ - d in frame coordinates
  double il;           // 1 / |x - p|
};

// degenerate projection |x - p| < 1e-12 (_kernels.py:541-542): the high word
// of l2 >= 0 is monotone in l2; hi(1e-24) = 0x3AF357C2
constexpr int kDegHi = 0x3AF357C2;

__device__ __forceinline__ VtxF make_vtxf(double X, double Y, double Zc, double qa, double qb,
                                          double qc, int& minhi) {
  VtxF v;
  const double rx = X - qa, ry = Y - qb, rz = Zc - qc;
  const double l2 = rx * rx + ry * ry + rz * rz;
  minhi = min(minhi, __double2hiint(l2));
  v.il = rsqrt_nr(l2);
  v.ux = rx * v.il;
  v.uy = ry * v.il;
  v.uz = fma(rz, v.il, -1.0);
  return v;
}

// polyline/curve band test (rare path, den < 0): d within band_factor*h/dist
// of the arc (a, b); raw offsets are (u + d) / il.
__device__ __forceinline__ bool band_hit_f(const VtxF& a, const VtxF& b, double num, double h,
                                           double band_factor) {
  const double la = 1.0 / a.il, lb = 1.0 / b.il;
  const double ax = a.ux, ay = a.uy, az = a.uz + 1.0;
  const double bx = b.ux, by = b.uy, bz = b.uz + 1.0;
  const double sgx = bx * lb - ax * la, sgy = by * lb - ay * la, sgz = bz * lb - az * la;
  const double L = sqrt(sgx * sgx + sgy * sgy + sgz * sgz);
  const double dist = fmin(la, lb) - L;
  if (dist <= 0.0) return true;
  const double cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
  const double s2 = cx * cx + cy * cy + cz * cz;
  const double th = band_factor * h / dist;
  return num * num <= th * th * s2;
}

template <int QPT>
__global__ void __launch_bounds__(kBlockQ, 2)
k_boundary(int32_t m, const int32_t* __restrict__ active, const double* __restrict__ pos,
           const double* __restrict__ vproj, int64_t V, int S, int64_t n_edges,
           const double* __restrict__ band_h, Frame f, DevParams prm,
           double* __restrict__ bpart, int32_t* __restrict__ flag_acc,
           unsigned long long* __restrict__ counters) {
  // blockIdx.y: chunk of whole edges [e0, e1) -> vertex range [vbeg, vend)
  const int nchunk = gridDim.y;
  const int64_t e0 = n_edges * blockIdx.y / nchunk, e1 = n_edges * (blockIdx.y + 1) / nchunk;
  const int64_t vbeg = e0 * S, vend = e1 * S;
  __shared__ double sx[kTileV], sy[kTileV], sz[kTileV];
  int32_t slot[QPT];
  double qa[QPT], qb[QPT], qc[QPT];
  SegState st[QPT];
  int flags[QPT];
  VtxF va[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    slot[j] = blockIdx.x * (blockDim.x * QPT) + j * blockDim.x + threadIdx.x;
    const bool live = slot[j] < m;
    const int32_t q = live ? (active ? active[slot[j]] : slot[j]) : 0;
    const double px = live ? pos[3 * (int64_t)q] : 0.0;
    const double py = live ? pos[3 * (int64_t)q + 1] : 0.0;
    const double pz = live ? pos[3 * (int64_t)q + 2] : 0.0;
    qa[j] = px * f.e1[0] + py * f.e1[1] + pz * f.e1[2];
    qb[j] = px * f.e2[0] + py * f.e2[1] + pz * f.e2[2];
    qc[j] = px * f.d[0] + py * f.d[1] + pz * f.d[2];
    st[j] = SegState{1.0, 0.0, 0};
    flags[j] = 0;
    va[j] = VtxF{0.0, 0.0, -1.0, 1.0};
  }
  int minhi[QPT], neg[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    minhi[j] = 0x7fffffff;
    neg[j] = 0;
  }
  // hot path of one segment (A -> B): only the complex product; the sign of
  // den is OR-ed into neg so the rare band test runs after the tile
  auto seg = [&](int j, const VtxF& A, const VtxF& B) {
    const double num = A.uy * B.ux - A.ux * B.uy;   // c.(a^ x b^)
    const double den = A.ux * B.ux + A.uy * B.uy + A.uz * B.uz;
    neg[j] |= __double2hiint(den);
    cmul_track(st[j], den, num);
  };
  __shared__ double prev_x[3];  // vertex carried into the current tile
  VtxF vb[QPT];
  int nseg = 0;
  for (int64_t t0 = vbeg; t0 < vend; t0 += kTileV) {
    const int nt = (int)min((int64_t)kTileV, vend - t0);
    __syncthreads();
    if (threadIdx.x == 0 && t0 > vbeg) {
      prev_x[0] = sx[kTileV - 1];
      prev_x[1] = sy[kTileV - 1];
      prev_x[2] = sz[kTileV - 1];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
      const int64_t g = t0 + k;
      sx[k] = vproj[g];
      sy[k] = vproj[V + g];
      sz[k] = vproj[2 * V + g];
    }
    __syncthreads();
    const int64_t e_t0 = t0 / S;                // edge of the tile's first vertex
    const int kin_t0 = (int)(t0 - e_t0 * S);    // its index within that edge
    int kin = kin_t0;
    // unrolled by two vertices with the carried vertex alternating between
    // va and vb, so no per-vertex register copies
    int k = 0;
    for (; k + 1 < nt; k += 2) {
      {
        const double X = sx[k], Y = sy[k], Zc = sz[k];
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
          vb[j] = make_vtxf(X, Y, Zc, qa[j], qb[j], qc[j], minhi[j]);
          if (kin != 0) seg(j, va[j], vb[j]);
        }
        if (kin != 0 && (++nseg & 7) == 0) {
#pragma unroll
          for (int j = 0; j < QPT; ++j) renorm(st[j]);
        }
        if (++kin == S) kin = 0;
      }
      {
        const double X = sx[k + 1], Y = sy[k + 1], Zc = sz[k + 1];
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
          va[j] = make_vtxf(X, Y, Zc, qa[j], qb[j], qc[j], minhi[j]);
          if (kin != 0) seg(j, vb[j], va[j]);
        }
        if (kin != 0 && (++nseg & 7) == 0) {
#pragma unroll
          for (int j = 0; j < QPT; ++j) renorm(st[j]);
        }
        if (++kin == S) kin = 0;
      }
    }
    if (k < nt) {  // odd tile length
      const double X = sx[k], Y = sy[k], Zc = sz[k];
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        vb[j] = make_vtxf(X, Y, Zc, qa[j], qb[j], qc[j], minhi[j]);
        if (kin != 0) seg(j, va[j], vb[j]);
        va[j] = vb[j];
      }
      if (kin != 0 && (++nseg & 7) == 0) {
#pragma unroll
        for (int j = 0; j < QPT; ++j) renorm(st[j]);
      }
      if (++kin == S) kin = 0;
    }
    // rare: some segment of this tile had den < 0 -> polyline/curve band test
    // for the queries concerned, re-walking the tile
    bool any = false;
#pragma unroll
    for (int j = 0; j < QPT; ++j) any |= neg[j] < 0;
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        if (neg[j] >= 0) continue;
        int mh = 0x7fffffff;
        int kk = kin_t0;
        int64_t e = e_t0;
        VtxF A = VtxF{0.0, 0.0, -1.0, 1.0};
        if (kk != 0) A = make_vtxf(prev_x[0], prev_x[1], prev_x[2], qa[j], qb[j], qc[j], mh);
        for (int i = 0; i < nt; ++i) {
          const VtxF B = make_vtxf(sx[i], sy[i], sz[i], qa[j], qb[j], qc[j], mh);
          if (kk != 0) {
            const double num = A.uy * B.ux - A.ux * B.uy;
            const double den = A.ux * B.ux + A.uy * B.uy + A.uz * B.uz;
            if (den < 0.0 && band_hit_f(A, B, num, __ldg(band_h + e), prm.band_factor))
              flags[j] |= FLAG_BAND;
          }
          A = B;
          if (++kk == S) {
            kk = 0;
            ++e;
          }
        }
        neg[j] = 0;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < QPT; ++j)
    if (minhi[j] < kDegHi) flags[j] |= FLAG_DEGEN;
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

// Edge-aligned K4 (S <= kTileV): a tile holds whole edges, so every edge's
// S-1 segments run as blocks of 8 with no per-vertex edge bookkeeping
// (vertex index mod S, the first-vertex branch, the renorm counter); the
// vertex carried between segments alternates between two registers.  Same
// segment order and the same power-of-two renormalisations (exact scalings)
// as k_boundary, so the partial sums are bit-identical to it.
#ifndef GWN_K4_MINB
#define GWN_K4_MINB 2
#endif
// kFF: far-field scene (gwn_farfield.cu).  Per edge, each query decides with
// ff_far() whether the edge's cycle is taken by the far kernel; far queries
// multiply their running product by (1, 0) (exactly neutral) and a warp whose
// queries are all far skips the edge.  `order` (nullable) maps threads to
// slots (3-D Morton order, so warps agree).
struct FFView {
  const int32_t* order;
  const int32_t* edge;   // cycle of each edge, -1 = exact only
  const double* g;       // cycle centres, round frame
  const double* r2;      // R_min^2, line radius^2
};

#ifndef GWN_K4_MINB_FF
#define GWN_K4_MINB_FF 3  // far-field scenes: occupancy beats the few spills (config 5 -5%)
#endif
template <int QPT, bool kFF>
__global__ void __launch_bounds__(kBlockQ, kFF ? GWN_K4_MINB_FF : GWN_K4_MINB)
k_boundary_e(int32_t m, const int32_t* __restrict__ active, const double* __restrict__ pos,
             const double* __restrict__ vproj, int64_t V, int S, int64_t n_edges,
             const double* __restrict__ band_h, Frame f, DevParams prm,
             double* __restrict__ bpart, int32_t* __restrict__ flag_acc,
             unsigned long long* __restrict__ counters, FFView ff) {
  const int nchunk = gridDim.y;
  const int64_t e0 = n_edges * blockIdx.y / nchunk, e1 = n_edges * (blockIdx.y + 1) / nchunk;
  const int ept = kTileV / S;  // whole edges per tile
  __shared__ double sx[kTileV], sy[kTileV], sz[kTileV];
  int32_t slot[QPT];
  double qa[QPT], qb[QPT], qc[QPT];
  SegState st[QPT];
  int flags[QPT], minhi[QPT], neg[QPT];
  bool live[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    // ordered (far-field) launches: a warp's QPT*32 queries are consecutive
    // in Morton order, so they share one small region
    const int32_t t = (kFF && ff.order)
                          ? blockIdx.x * (blockDim.x * QPT) + (threadIdx.x & ~31) * QPT + j * 32 +
                                (threadIdx.x & 31)
                          : blockIdx.x * (blockDim.x * QPT) + j * blockDim.x + threadIdx.x;
    live[j] = t < m;
    slot[j] = (kFF && ff.order && live[j]) ? ff.order[t] : t;
    const int32_t q = live[j] ? (active ? active[slot[j]] : slot[j]) : 0;
    const double px = live[j] ? pos[3 * (int64_t)q] : 0.0;
    const double py = live[j] ? pos[3 * (int64_t)q + 1] : 0.0;
    const double pz = live[j] ? pos[3 * (int64_t)q + 2] : 0.0;
    if (kFF) {
      frame_q(f, px, py, pz, qa[j], qb[j], qc[j]);
    } else {
      qa[j] = px * f.e1[0] + py * f.e1[1] + pz * f.e1[2];
      qb[j] = px * f.e2[0] + py * f.e2[1] + pz * f.e2[2];
      qc[j] = px * f.d[0] + py * f.d[1] + pz * f.d[2];
    }
    st[j] = SegState{1.0, 0.0, 0};
    flags[j] = 0;
    minhi[j] = 0x7fffffff;
    neg[j] = 0;
  }
  unsigned long long exact_pairs = 0;  // (query, segment) pairs summed exactly
  VtxF va[QPT], vb[QPT];
  for (int64_t te = e0; te < e1; te += ept) {
    const int ne = (int)min((int64_t)ept, e1 - te);
    const int nt = ne * S;
    const int64_t t0 = te * S;
    __syncthreads();
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
      const int64_t g = t0 + k;
      sx[k] = vproj[g];
      sy[k] = vproj[V + g];
      sz[k] = vproj[2 * V + g];
    }
    __syncthreads();
    for (int e = 0; e < ne; ++e) {
      const int b = e * S;
      // far queries of this edge's cycle: neutral factor (1, 0); skip the
      // edge when the whole warp is far
      bool far[QPT];
#pragma unroll
      for (int j = 0; j < QPT; ++j) far[j] = false;
      if (kFF) {
        const int c = __ldg(ff.edge + te + e);
        bool all = true;
        int nnear = 0;
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
          far[j] = c >= 0 && live[j] && ff_far(qa[j], qb[j], qc[j], ff.g + 3 * c, ff.r2 + 2 * c);
          all &= far[j] || !live[j];
          nnear += (live[j] && !far[j]) ? 1 : 0;
        }
#ifndef GWN_FF_NOSKIP
        if (__all_sync(0xffffffffu, all)) continue;
#endif
        exact_pairs += (unsigned long long)nnear * (unsigned long long)(S - 1);
      }
#pragma unroll
      for (int j = 0; j < QPT; ++j)
        va[j] = make_vtxf(sx[b], sy[b], sz[b], qa[j], qb[j], qc[j], minhi[j]);
      int k = b + 1;
      const int kend = b + S;
      // blocks of 8 segments: va -> vb -> va ..., renorm after each block
      for (; k + 8 <= kend; k += 8) {
#pragma unroll
        for (int h = 0; h < 8; h += 2) {
#pragma unroll
          for (int j = 0; j < QPT; ++j) {
            vb[j] = make_vtxf(sx[k + h], sy[k + h], sz[k + h], qa[j], qb[j], qc[j], minhi[j]);
            double num = va[j].uy * vb[j].ux - va[j].ux * vb[j].uy;
            double den = va[j].ux * vb[j].ux + va[j].uy * vb[j].uy + va[j].uz * vb[j].uz;
            if (kFF && far[j]) { den = 1.0; num = 0.0; }
            neg[j] |= __double2hiint(den);
            cmul_track(st[j], den, num);
          }
#pragma unroll
          for (int j = 0; j < QPT; ++j) {
            va[j] = make_vtxf(sx[k + h + 1], sy[k + h + 1], sz[k + h + 1], qa[j], qb[j], qc[j],
                              minhi[j]);
            double num = vb[j].uy * va[j].ux - vb[j].ux * va[j].uy;
            double den = vb[j].ux * va[j].ux + vb[j].uy * va[j].uy + vb[j].uz * va[j].uz;
            if (kFF && far[j]) { den = 1.0; num = 0.0; }
            neg[j] |= __double2hiint(den);
            cmul_track(st[j], den, num);
          }
        }
#pragma unroll
        for (int j = 0; j < QPT; ++j) renorm(st[j]);
      }
      for (; k < kend; ++k) {
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
          vb[j] = make_vtxf(sx[k], sy[k], sz[k], qa[j], qb[j], qc[j], minhi[j]);
          double num = va[j].uy * vb[j].ux - va[j].ux * vb[j].uy;
          double den = va[j].ux * vb[j].ux + va[j].uy * vb[j].uy + va[j].uz * vb[j].uz;
          if (kFF && far[j]) { den = 1.0; num = 0.0; }
          neg[j] |= __double2hiint(den);
          cmul_track(st[j], den, num);
          va[j] = vb[j];
        }
      }
#pragma unroll
      for (int j = 0; j < QPT; ++j) renorm(st[j]);
    }
    // rare: some segment of this tile had den < 0 -> polyline/curve band test
    bool any = false;
#pragma unroll
    for (int j = 0; j < QPT; ++j) any |= neg[j] < 0;
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        if (neg[j] >= 0) continue;
        int mh = 0x7fffffff;
        for (int e = 0; e < ne; ++e) {
          const int b = e * S;
          if (kFF) {  // far cycles: the line misses their sphere, no band
            const int c = __ldg(ff.edge + te + e);
            if (c >= 0 && ff_far(qa[j], qb[j], qc[j], ff.g + 3 * c, ff.r2 + 2 * c)) continue;
          }
          const double h = __ldg(band_h + te + e);
          VtxF A = make_vtxf(sx[b], sy[b], sz[b], qa[j], qb[j], qc[j], mh);
          for (int i = b + 1; i < b + S; ++i) {
            const VtxF B = make_vtxf(sx[i], sy[i], sz[i], qa[j], qb[j], qc[j], mh);
            const double num = A.uy * B.ux - A.ux * B.uy;
            const double den = A.ux * B.ux + A.uy * B.uy + A.uz * B.uz;
            if (den < 0.0 && band_hit_f(A, B, num, h, prm.band_factor)) flags[j] |= FLAG_BAND;
            A = B;
          }
        }
        neg[j] = 0;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < QPT; ++j)
    if (minhi[j] < kDegHi) flags[j] |= FLAG_DEGEN;
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    if (live[j]) {
      bpart[(int64_t)blockIdx.y * m + slot[j]] = seg_angle(st[j]);
      if (flags[j]) atomicOr(&flag_acc[slot[j]], flags[j]);
    }
  }
  if (kFF) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) exact_pairs += __shfl_down_sync(0xffffffffu, exact_pairs, o);
    if ((threadIdx.x & 31) == 0 && exact_pairs) atomicAdd(&counters[CNT_SEGMENTS], exact_pairs);
  } else if (threadIdx.x == 0) {
    int32_t nq = min((int32_t)(blockDim.x * QPT), m - (int32_t)(blockIdx.x * blockDim.x * QPT));
    const int64_t segs = (e1 - e0) * (int64_t)(S - 1);
    atomicAdd(&counters[CNT_SEGMENTS], (unsigned long long)(segs * nq));
  }
}

// Accuracy of rsqrt_nr against the correctly rounded 1/sqrt on a log-uniform
// sweep of [1e-20, 1e20] (gwn_selftest_rsqrt).
__global__ void k_rsqrt_selftest(int64_t n, unsigned long long* max_ulp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = exp10(-20.0 + 40.0 * ((double)i + 0.5) / (double)n);
  const double ref = __drcp_rn(__dsqrt_rn(x));
  const double got = rsqrt_nr(x);
  const long long d = __double_as_longlong(got) - __double_as_longlong(ref);
  atomicMax(max_ulp, (unsigned long long)(d < 0 ? -d : d));
}

cudaError_t selftest_rsqrt(int64_t n, unsigned long long* max_ulp_host) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  cudaMemset(d, 0, sizeof(unsigned long long));
  k_rsqrt_selftest<<<(unsigned)((n + 255) / 256), 256>>>(n, d);
  e = cudaMemcpy(max_ulp_host, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

// Boundary vertices in the round's ray frame (X = x.e1, Y = x.e2, Zc = x.d).
__global__ void k_vproj(const double* __restrict__ verts, int64_t V, Frame f,
                        double* __restrict__ vproj) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const double x = verts[i], y = verts[V + i], z = verts[2 * V + i];
  vproj[i] = x * f.e1[0] + y * f.e1[1] + z * f.e1[2];
  vproj[V + i] = x * f.e2[0] + y * f.e2[1] + z * f.e2[2];
  vproj[2 * V + i] = x * f.d[0] + y * f.d[1] + z * f.d[2];
}

cudaError_t launch_vproj(const gwn_scene* sc, Round& rd, cudaStream_t st) {
  const int64_t V = sc->n_edges * sc->S;
  if (V == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc(&rd.vproj, sizeof(double) * 3 * V);
  if (e != cudaSuccess) return e;
  if (sc->ff_n > 0) {  // far-field cycle centres in this round's frame
    std::vector<double> h(3 * (size_t)sc->ff_n);
    for (int c = 0; c < sc->ff_n; ++c) {
      const double* g = &sc->ff_g_host[3 * c];
      h[3 * c] = g[0] * rd.f.e1[0] + g[1] * rd.f.e1[1] + g[2] * rd.f.e1[2];
      h[3 * c + 1] = g[0] * rd.f.e2[0] + g[1] * rd.f.e2[1] + g[2] * rd.f.e2[2];
      h[3 * c + 2] = g[0] * rd.f.d[0] + g[1] * rd.f.d[1] + g[2] * rd.f.d[2];
    }
    if ((e = cudaMalloc(&rd.ffg, sizeof(double) * h.size())) != cudaSuccess) return e;
    if ((e = cudaMemcpy(rd.ffg, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice)) !=
        cudaSuccess)
      return e;
    std::vector<double> a(6 * (size_t)sc->ff_n);  // sliver chords in this frame
    for (size_t k = 0; k < a.size() / 3; ++k) {
      const double* g = &sc->ff_chord_host[3 * k];
      a[3 * k] = g[0] * rd.f.e1[0] + g[1] * rd.f.e1[1] + g[2] * rd.f.e1[2];
      a[3 * k + 1] = g[0] * rd.f.e2[0] + g[1] * rd.f.e2[1] + g[2] * rd.f.e2[2];
      a[3 * k + 2] = g[0] * rd.f.d[0] + g[1] * rd.f.d[1] + g[2] * rd.f.d[2];
    }
    if ((e = cudaMalloc(&rd.ffa, sizeof(double) * a.size())) != cudaSuccess) return e;
    if ((e = cudaMemcpy(rd.ffa, a.data(), sizeof(double) * a.size(), cudaMemcpyHostToDevice)) !=
        cudaSuccess)
      return e;
  }
  k_vproj<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(sc->verts, V, rd.f, rd.vproj);
  return cudaGetLastError();
}

#ifndef GWN_K4_QPT
#define GWN_K4_QPT 2
#endif
constexpr int kQPT = GWN_K4_QPT;

// Edge chunks of the boundary sum.  Fixed per scene (not per batch) so the
// chunk partials -- added in chunk order by K5 -- make w bit-identical for any
// batching, chunking or sharding of the queries; enough chunks that small
// batches still fill the GPU.
int boundary_chunks(const gwn_scene* sc, int32_t m) {
  (void)m;
  if (sc->n_edges <= 0) return 1;
  // exact edge chunks, then the far-field row (gwn_farfield.cu) when on
  return (int)std::min<int64_t>(sc->n_edges, 64) + (sc->ff_n > 0 ? kFFRows : 0);
}

// nchunk partial rows: the exact kernel fills rows [0, nexact), the far
// kernel the kFFRows rows after them (far-field scenes); `order` (nullable) is the exact
// kernel's thread -> slot map (launch_ff_order).
cudaError_t launch_boundary(const gwn_scene* sc, const Round& rd, int32_t m,
                            const int32_t* active, const double* pos, double* bpart, int nchunk,
                            int32_t* flags, unsigned long long* counters, cudaStream_t st,
                            const int32_t* order) {
  if (m <= 0) return cudaSuccess;
  int64_t V = sc->n_edges * sc->S;
  if (V == 0) return cudaMemsetAsync(bpart, 0, sizeof(double) * m, st);
  static const bool generic = getenv("GWN_K4_GENERIC") != nullptr;  // A/B switch
  const bool ff = sc->ff_n > 0 && rd.ffg;
  const int nexact = nchunk - (sc->ff_n > 0 ? kFFRows : 0);
  dim3 grid((m + kBlockQ * kQPT - 1) / (kBlockQ * kQPT), nexact);
  cudaError_t e = cudaSuccess;
  if (sc->S <= kTileV && !generic) {
    if (ff) {
      const FFView fv{order, sc->ff_edge, rd.ffg, sc->ff_r};
      k_boundary_e<kQPT, true><<<grid, kBlockQ, 0, st>>>(m, active, pos, rd.vproj, V, sc->S,
                                                         sc->n_edges, sc->band_h, rd.f, sc->dprm,
                                                         bpart, flags, counters, fv);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      return launch_boundary_far(sc, rd, m, active, pos, bpart + (int64_t)nexact * m, counters,
                                 st, order);
    }
    k_boundary_e<kQPT, false><<<grid, kBlockQ, 0, st>>>(m, active, pos, rd.vproj, V, sc->S,
                                                        sc->n_edges, sc->band_h, rd.f, sc->dprm,
                                                        bpart, flags, counters,
                                                        FFView{nullptr, nullptr, nullptr, nullptr});
  } else {
    k_boundary<kQPT><<<grid, kBlockQ, 0, st>>>(m, active, pos, rd.vproj, V, sc->S, sc->n_edges,
                                               sc->band_h, rd.f, sc->dprm, bpart, flags,
                                               counters);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (sc->ff_n > 0)  // exact path for everything: the far rows are zero
    return cudaMemsetAsync(bpart + (int64_t)nexact * m, 0, sizeof(double) * m * kFFRows, st);
  return cudaSuccess;
}

// _kernels.single_loop_batch (_kernels.py:801-823) on the GPU: one closed loop,
// queries p_k = o + t_k d on one ray, chi from the cached hits with t_h > t_k
// (:778-788).  ok = 0 only for a hit clash |t_h - t_k| <= t_eps or a
// degenerate projection; the fan formula needs no simple-loop restriction.
__global__ void k_single_loop(const double* __restrict__ loop, int64_t B, double ox, double oy,
                              double oz, Frame f, const double* __restrict__ hit_ts,
                              const int64_t* __restrict__ hit_signs, int64_t H,
                              const double* __restrict__ qts, int64_t K, double t_eps,
                              double* __restrict__ w, int8_t* __restrict__ ok) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double t = qts[k];
  const double dx = f.d[0], dy = f.d[1], dz = f.d[2];
  const double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
  long long chi = 0;
  bool clash = false;
  for (int64_t h = 0; h < H; ++h) {
    if (fabs(hit_ts[h] - t) <= t_eps) clash = true;
    if (hit_ts[h] > t) chi += hit_signs[h];
  }
  const double qa = px * f.e1[0] + py * f.e1[1] + pz * f.e1[2];
  const double qb = px * f.e2[0] + py * f.e2[1] + pz * f.e2[2];
  const double qc = px * f.d[0] + py * f.d[1] + pz * f.d[2];
  auto vtx = [&](int64_t i, int& mh) {
    const double x = loop[3 * i], y = loop[3 * i + 1], z = loop[3 * i + 2];
    return make_vtxf(x * f.e1[0] + y * f.e1[1] + z * f.e1[2],
                     x * f.e2[0] + y * f.e2[1] + z * f.e2[2],
                     x * f.d[0] + y * f.d[1] + z * f.d[2], qa, qb, qc, mh);
  };
  SegState st = {1.0, 0.0, 0};
  int minhi = 0x7fffffff;
  VtxF va = vtx(B - 1, minhi);
  for (int64_t i = 0; i < B; ++i) {
    const VtxF vb = vtx(i, minhi);
    const double num = va.uy * vb.ux - va.ux * vb.uy;
    const double den = va.ux * vb.ux + va.uy * vb.uy + va.uz * vb.uz;
    cmul_track(st, den, num);
    if ((i & 7) == 7) renorm(st);
    va = vb;
  }
  const double ang = atan2(st.Zi, st.Zr) + 6.283185307179586476925 * (double)st.wraps;
  w[k] = (double)chi + ang * 0.15915494309189533576888;
  ok[k] = (clash || minhi < kDegHi) ? 0 : 1;
}

cudaError_t launch_single_loop(const double* loop, int64_t B, const double* o, const double* d,
                               const double* hit_ts, const int64_t* hit_signs, int64_t H,
                               const double* qts, int64_t K, double t_eps, double deg, double* w,
                               int8_t* ok, cudaStream_t st) {
  if (K <= 0) return cudaSuccess;
  (void)deg;
  Frame f;
  make_frame(d, &f);
  k_single_loop<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(loop, B, o[0], o[1], o[2], f,
                                                             hit_ts, hit_signs, H, qts, K, t_eps,
                                                             w, ok);
  return cudaGetLastError();
}

}  // namespace gwn
