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

#include <cub/cub.cuh>

#include "gwn_fan.cuh"
#include "gwn_farfield.cuh"

namespace gwn {

constexpr int kTileV = 2000;   // vertices per shared-memory tile (3 x 2000 x 8 B = 48 KB)
constexpr int kBlockQ = 256;   // queries (threads) per block

// Per-vertex quantities of the shifted fan formula in the round's ray frame
// (e1, e2, d): d = (0,0,1).  The segment factor den + i num is used only
// through its argument, so it may carry any positive scale: with the raw
// offsets r_a = a - p, l_a = |r_a| and u_a = r_a - l_a d (= l_a (a^ - d)),
//     den' = u_a . u_b = l_a l_b (1 + a^.b^ + b^.c + c.a^),
//     num' = u_a,y u_b,x - u_a,x u_b,y = l_a l_b c.(a^ x b^),
// the same expressions as for the unit vectors without the three
// normalising multiplications per vertex (2 of 23 FP64 operations per
// segment).  The running product is renormalised (exact power of two) every
// 8 segments; coordinates up to ~1e18 stay far from overflow.
#ifndef GWN_K4_UNNORM
#define GWN_K4_UNNORM 1
#endif
struct VtxF {
  double ux, uy, uz;   // GWN_K4_UNNORM: r - l d, else a^ - d (frame coordinates)
  double il;           // GWN_K4_UNNORM: l = |x - p|, else 1 / |x - p|
};

// degenerate projection |x - p| < 1e-12 (_kernels.py:541-542): the high word
// of l2 >= 0 is monotone in l2; hi(1e-24) = 0x3AF357C2
constexpr int kDegHi = 0x3AF357C2;

// sqrt(x) to full precision from the MUFU.RSQ64H seed y (~2^-22): with
// h = x y and e = 1 - x y^2, sqrt(x) = h (1 - e)^(-1/2) = h (1 + e/2 + 3e^2/8)
// (the companion of rsqrt_nr; no special-value path, see there)
__device__ __forceinline__ double sqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = x * y;
  const double e = fma(-h, y, 1.0);
  const double p = fma(0.375, e, 0.5);
  return fma(h * e, p, h);
}

__device__ __forceinline__ VtxF make_vtxf(double X, double Y, double Zc, double qa, double qb,
                                          double qc, int& minhi) {
  VtxF v;
  const double rx = X - qa, ry = Y - qb, rz = Zc - qc;
  const double l2 = rx * rx + ry * ry + rz * rz;
  minhi = min(minhi, __double2hiint(l2));
#if GWN_K4_UNNORM
  v.il = sqrt_nr(l2);
  v.ux = rx;
  v.uy = ry;
  v.uz = rz - v.il;
#else
  v.il = rsqrt_nr(l2);
  v.ux = rx * v.il;
  v.uy = ry * v.il;
  v.uz = fma(rz, v.il, -1.0);
#endif
  return v;
}

// polyline/curve band test (rare path, den < 0): d within band_factor*h/dist
// of the arc (a, b); `num` is the segment's num as computed from a and b (it
// carries the scale l_a l_b under GWN_K4_UNNORM, and so does the cross
// product below: the test is the same).
__device__ __forceinline__ bool band_hit_f(const VtxF& a, const VtxF& b, double num, double h,
                                           double band_factor) {
#if GWN_K4_UNNORM
  const double la = a.il, lb = b.il;
  const double ax = a.ux, ay = a.uy, az = a.uz + la;   // raw offsets
  const double bx = b.ux, by = b.uy, bz = b.uz + lb;
  const double sgx = bx - ax, sgy = by - ay, sgz = bz - az;
#else
  const double la = 1.0 / a.il, lb = 1.0 / b.il;
  const double ax = a.ux, ay = a.uy, az = a.uz + 1.0;
  const double bx = b.ux, by = b.uy, bz = b.uz + 1.0;
  const double sgx = bx * lb - ax * la, sgy = by * lb - ay * la, sgz = bz * lb - az * la;
#endif
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

// one edge's S-1 segments from shared memory (vertex b .. b+S-1) into the
// running products: blocks of 8 segments, renormalised after each block
template <int QPT>
__device__ __forceinline__ void edge_segments(const double* sx, const double* sy,
                                              const double* sz, int b, int S, const bool* use,
                                              const double* qa, const double* qb,
                                              const double* qc, SegState* st, int* neg,
                                              int* minhi, VtxF* va, VtxF* vb) {
#pragma unroll
  for (int j = 0; j < QPT; ++j)
    va[j] = make_vtxf(sx[b], sy[b], sz[b], qa[j], qb[j], qc[j], minhi[j]);
  int k = b + 1;
  const int kend = b + S;
  for (; k + 8 <= kend; k += 8) {
#pragma unroll
    for (int h = 0; h < 8; h += 2) {
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        vb[j] = make_vtxf(sx[k + h], sy[k + h], sz[k + h], qa[j], qb[j], qc[j], minhi[j]);
        const double num = va[j].uy * vb[j].ux - va[j].ux * vb[j].uy;
        const double den = va[j].ux * vb[j].ux + va[j].uy * vb[j].uy + va[j].uz * vb[j].uz;
        neg[j] |= __double2hiint(den);
        cmul_track(st[j], den, num);
      }
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        va[j] = make_vtxf(sx[k + h + 1], sy[k + h + 1], sz[k + h + 1], qa[j], qb[j], qc[j],
                          minhi[j]);
        const double num = vb[j].uy * va[j].ux - vb[j].ux * va[j].uy;
        const double den = vb[j].ux * va[j].ux + vb[j].uy * va[j].uy + vb[j].uz * va[j].uz;
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
      const double num = va[j].uy * vb[j].ux - va[j].ux * vb[j].uy;
      const double den = va[j].ux * vb[j].ux + va[j].uy * vb[j].uy + va[j].uz * vb[j].uz;
      neg[j] |= __double2hiint(den);
      cmul_track(st[j], den, num);
      va[j] = vb[j];
    }
  }
#pragma unroll
  for (int j = 0; j < QPT; ++j) renorm(st[j]);
  (void)use;
}

// Some segment of the staged edges had den < 0 for some lane: polyline/curve
// band test for the lanes concerned.  Warp-cooperative: a flagged lane's
// query is broadcast and the 32 lanes share the staged segments (each segment
// with the same operations a single lane would use, so the flags are the
// same).  One lane re-walking every staged edge alone while 31 wait was 12% of
// k_ff_near's issued instructions at config 5 (ncu: 28.3 active threads per
// warp).  Every lane of the warp must call this.
template <int QPT>
__device__ __forceinline__ void band_rewalk(const double* sx, const double* sy, const double* sz,
                                            int ne, int S, const double* __restrict__ band_h,
                                            int64_t e_first, const double* qa, const double* qb,
                                            const double* qc, double band_factor, int* neg,
                                            int* flags) {
  bool any = false;
#pragma unroll
  for (int j = 0; j < QPT; ++j) any |= neg[j] < 0;
  if (!__any_sync(0xffffffffu, any)) return;
  const int lane = threadIdx.x & 31;
  const int spe = S - 1, nseg = ne * spe;  // segments per edge, staged segments
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    unsigned need = __ballot_sync(0xffffffffu, neg[j] < 0);
    while (need) {
      const int src = __ffs(need) - 1;
      need &= need - 1;
      const double a = __shfl_sync(0xffffffffu, qa[j], src);
      const double b = __shfl_sync(0xffffffffu, qb[j], src);
      const double c = __shfl_sync(0xffffffffu, qc[j], src);
      bool hit = false;
      int mh = 0x7fffffff;
      for (int t = lane; t < nseg; t += 32) {
        const int e = t / spe, i = e * S + (t - e * spe);  // segment (i, i + 1) of edge e
        const VtxF A = make_vtxf(sx[i], sy[i], sz[i], a, b, c, mh);
        const VtxF B = make_vtxf(sx[i + 1], sy[i + 1], sz[i + 1], a, b, c, mh);
        const double num = A.uy * B.ux - A.ux * B.uy;
        const double den = A.ux * B.ux + A.uy * B.uy + A.uz * B.uz;
        if (den < 0.0 && band_hit_f(A, B, num, __ldg(band_h + e_first + e), band_factor))
          hit = true;
      }
      if (__any_sync(0xffffffffu, hit) && lane == src) flags[j] |= FLAG_BAND;
    }
    neg[j] = 0;
  }
}

template <int QPT>
__global__ void __launch_bounds__(kBlockQ, GWN_K4_MINB)
k_boundary_e(int32_t m, const int32_t* __restrict__ active, const double* __restrict__ pos,
             const double* __restrict__ vproj, int64_t V, int S, int64_t n_edges,
             const double* __restrict__ band_h, Frame f, DevParams prm,
             double* __restrict__ bpart, int32_t* __restrict__ flag_acc,
             unsigned long long* __restrict__ counters) {
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
    const int32_t t = blockIdx.x * (blockDim.x * QPT) + j * blockDim.x + threadIdx.x;
    live[j] = t < m;
    slot[j] = t;
    const int32_t q = live[j] ? (active ? active[slot[j]] : slot[j]) : 0;
    const double px = live[j] ? pos[3 * (int64_t)q] : 0.0;
    const double py = live[j] ? pos[3 * (int64_t)q + 1] : 0.0;
    const double pz = live[j] ? pos[3 * (int64_t)q + 2] : 0.0;
    qa[j] = px * f.e1[0] + py * f.e1[1] + pz * f.e1[2];
    qb[j] = px * f.e2[0] + py * f.e2[1] + pz * f.e2[2];
    qc[j] = px * f.d[0] + py * f.d[1] + pz * f.d[2];
    st[j] = SegState{1.0, 0.0, 0};
    flags[j] = 0;
    minhi[j] = 0x7fffffff;
    neg[j] = 0;
  }
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
    for (int e = 0; e < ne; ++e)
      edge_segments<QPT>(sx, sy, sz, e * S, S, live, qa, qb, qc, st, neg, minhi, va, vb);
    band_rewalk<QPT>(sx, sy, sz, ne, S, band_h, te, qa, qb, qc, prm.band_factor, neg, flags);
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
  if (threadIdx.x == 0) {
    int32_t nq = min((int32_t)(blockDim.x * QPT), m - (int32_t)(blockIdx.x * blockDim.x * QPT));
    const int64_t segs = (e1 - e0) * (int64_t)(S - 1);
    atomicAdd(&counters[CNT_SEGMENTS], (unsigned long long)(segs * nq));
  }
}

#ifndef GWN_K4_QPT
#define GWN_K4_QPT 2
#endif
constexpr int kQPT = GWN_K4_QPT;
// the far-field scenes' exact kernel (k_ff_near): one pair per thread at four
// 256-thread blocks per SM (config 5 at 2^24: 111.6 -> 104.1 ms against
// two pairs per thread at two blocks; tools/k4_variants.py)
constexpr int kNearQPT = 1;
#ifndef GWN_NEAR_MINB
#define GWN_NEAR_MINB 4
#endif
constexpr int kNearMinBlocks = GWN_NEAR_MINB;

// ---------------------------------------------------------------------------
// Far-field scenes (entries built by gwn_farfield.cu).  Per round and chunk:
//   k_ff_count   per query (3-D Morton order), every entry: far or near?
//                counts per query and per entry (warp-aggregated atomics)
//   scans        query-major offsets qoff, entry-major offsets eoff, tiles
//   k_ff_fill    the same decisions again: far entries add their multipole
//                expansion (row 0), near ones append (query slot, k) to the
//                entry's pair list
//   k_ff_near    one block per tile of one entry's near pairs: the entry's
//                vertices staged once in shared memory, every lane sums the
//                exact fan over all of the entry's segments for its query --
//                no lane is ever masked, unlike a query-major walk over all
//                edges that skips far entries per lane
//   k_ff_near_sum  per query: its near angles in entry order (row 1)
// Both rows and every sum in them are in a fixed order, so w is
// bit-identical for any batching, chunking or sharding.
//
// Far test (both passes, bit-identical): R >= R_min(entry) and the ray's
// forward half-line p + t d (t > 0) misses the entry's sphere -- the fan sum's
// 2 pi branch sits where +d meets the polyline, so only that half-line
// matters (a sphere wholly behind p along d is far even when the backward
// line crosses it).
// ---------------------------------------------------------------------------

// Shadow winding grids (per round and closed expanded cycle): a pair whose
// forward half-line crosses the cycle's sphere, with the sphere wholly in
// front of the query, is far too when its cell is clean -- its exact fan sum
// is then the expansion's value plus kShadowJump times the winding number of
// the cycle's projection along d around the query (k_ff_wind).
constexpr int kWG = 128;             // cells per side over the sphere's disk
constexpr int kWDirty = -128;        // a cell some segment may come near
#ifndef GWN_SHADOW_SIGN
#define GWN_SHADOW_SIGN -1
#endif
// in the units of the far rows (Omega; halved into the partial angle sums)
constexpr double kShadowJump = GWN_SHADOW_SIGN * 12.566370614359172954;

struct FFRound {
  int32_t C;
  const double* g3;     // (C,3) entry centres in the round frame
  const double* r2;     // (C,2) R_min^2, line radius^2
  const double* lv;     // (C,kFFLevels) R^2 thresholds of the orders
  const double* gw;     // (C,3) entry centres (world)
  const double2* D;     // (C,kFFTerms) moments
  const int32_t* chord; // (C) sliver chord edge or -1
  const double* ffa;    // (C,6) chord end points, round frame
  const int8_t* wg;     // (C,kWG,kWG) shadow winding grids (k_ff_wind)
  const double* wgeo;   // (C,3) grid origin and inverse cell size
};

// Far test of entry c (every pass calls it on the same bits, so the
// decisions agree): 0 = near (the exact fan sum); 1 = far, R >= R_min and the
// forward half-line misses the entry's sphere (wind = 0); 2 = far, R >= R_min,
// the half-line crosses the sphere and the query's cell of the entry's shadow
// winding grid is clean (wind = the cell's value; see k_ff_wind).
__device__ __forceinline__ int ff_class(const FFRound& R, int32_t c, double qa, double qb,
                                        double qc, int& wind) {
  const double* g3 = R.g3 + 3 * (int64_t)c;
  const double* r2 = R.r2 + 2 * (int64_t)c;
  const double dx = __dsub_rn(__ldg(g3), qa), dy = __dsub_rn(__ldg(g3 + 1), qb);
  const double dz = __dsub_rn(__ldg(g3 + 2), qc);
  const double l2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  const double R2 = __dadd_rn(l2, __dmul_rn(dz, dz));
  const double line2 = __ldg(r2 + 1);
  wind = 0;
  if (!(R2 > __ldg(r2))) return 0;
  if (l2 > line2 || (dz < 0.0 && __dmul_rn(dz, dz) > line2)) return 1;
  // the forward half-line crosses the sphere, which lies wholly in front of
  // the query (R > R_min > the sphere's radius)
#ifdef GWN_NO_SHADOW
  return 0;
#endif
  const double* gg = R.wgeo + 3 * (int64_t)c;
  const double fx = __dmul_rn(__dsub_rn(qa, __ldg(gg)), __ldg(gg + 2));
  const double fy = __dmul_rn(__dsub_rn(qb, __ldg(gg + 1)), __ldg(gg + 2));
  if (!(fx >= 0.0 && fx < (double)kWG && fy >= 0.0 && fy < (double)kWG)) return 0;
  const int v = __ldg(R.wg + ((int64_t)c * kWG + (int)fy) * kWG + (int)fx);
  if (v == kWDirty) return 0;
  wind = v;
  return 2;
}

// Clenshaw coefficients of the irregular-harmonic recurrence (2n+1, (n+1)^2)
struct FFClen {
  double a[kFFK + 1], sq[kFFK + 2];
};
__constant__ FFClen c_ffc;

cudaError_t ff_init_constants() {  // per device, before the first far-field launch
  FFClen h;
  for (int n = 0; n <= kFFK; ++n) h.a[n] = 2.0 * n + 1.0;
  for (int n = 0; n <= kFFK + 1; ++n) h.sq[n] = (double)n * (double)n;
  return cudaMemcpyToSymbol(c_ffc, &h, sizeof h);
}

// Omega(p) = -sum_{n>=1} [Re(D_n^0 I_n^0) + 2 sum_{m>=1} Re(D_n^m I_n^m)] of
// order P.  Per column m, Clenshaw's backward sum over the three-term
// recurrence I_{n+1}^m = alpha_n I_n^m + beta_n I_{n-1}^m
// (alpha_n = (2n+1) z / r^2, beta_n = (m^2 - n^2) / r^2):
//     b_n = D_n^m + alpha_n b_{n+1} + beta_{n+1} b_{n+2},  sum = b_m I_m^m,
// six FP64 operations per term (the forward recurrence took ten); checked
// against the forward sum to 7e-15 relative at 2.4 cycle radii
// (tools/farfield/fmm_proto.py).  Column m = 0 starts at n = 1 (n = 0 has no
// moment): its sum is b_1 I_1^0 + beta_1 b_2 I_0^0 with beta_1 = -1/r^2.
// ff_eval_own runs four columns m at a time: they share the loop, the loads
// of the recurrence constants and alpha_n, and give the FP64 pipe four
// independent chains.  Every column's operations and their order depend only
// on (P, m), and the columns are added in increasing m, so a pair's value is
// the same bits in every kernel that evaluates it (warp-per-query rounds and
// the bucketed far pairs).
struct FFCol {
  double b1R, b1I, b2R, b2I;
};

__device__ __forceinline__ void ff_col_step(FFCol& c, double2 d, double al, double be) {
  const double bR = __fma_rn(al, c.b1R, __fma_rn(be, c.b2R, d.x));
  const double bI = __fma_rn(al, c.b1I, __fma_rn(be, c.b2I, d.y));
  c.b2R = c.b1R;
  c.b2I = c.b1I;
  c.b1R = bR;
  c.b1I = bI;
}

__device__ __forceinline__ double ff_eval_own(double x, double y, double z,
                                              const double2* Dc, int P) {
  const double ir2 = __drcp_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)),
                                         __dmul_rn(z, z)));
  const double zr = __dmul_rn(z, ir2);
  double dR = __dsqrt_rn(ir2), dI = 0.0;  // I_m^m of the next column
  double acc = 0.0;
#pragma unroll 1
  for (int m0 = 0; m0 <= P; m0 += 4) {
    FFCol col[4];
    double m2r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      col[i] = FFCol{0.0, 0.0, 0.0, 0.0};
      m2r[i] = __dmul_rn(c_ffc.sq[min(m0 + i, kFFK + 1)], ir2);  // (m0 + i)^2 from the table
    }
    // n from P down to m0 + 3: all four columns (when they exist)
    const int nall = m0 + 3;
    const double2* dp = Dc + ff_term(P, m0);
#pragma unroll 2
    for (int n = P; n >= nall; --n) {
      const double al = __dmul_rn(c_ffc.a[n], zr);
      const double sq = c_ffc.sq[n + 1];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        ff_col_step(col[i], dp[i], al, __fma_rn(-sq, ir2, m2r[i]));
      dp -= n;
    }
    // the tail: column m0 + i ends at n = m0 + i (n = 0 has no moment)
#pragma unroll
    for (int t = 2; t >= 0; --t) {
      const int n = m0 + t;
      if (n > P || n < 1) continue;
      const double al = __dmul_rn(c_ffc.a[n], zr);
      const double sq = c_ffc.sq[n + 1];
      const double2* dn = Dc + ff_term(n, m0);
#pragma unroll
      for (int i = 0; i <= t; ++i)
        ff_col_step(col[i], dn[i], al, __fma_rn(-sq, ir2, m2r[i]));
    }
    // column sums in increasing m
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int mm = m0 + i;
      if (mm > P) break;
      if (mm > 0) {  // I_m^m = -(2m-1)(x+iy)/r^2 I_{m-1}^{m-1}
        const double c0 = __dmul_rn(-c_ffc.a[mm - 1], ir2);  // -(2 mm - 1) from the table
        const double nR = __dmul_rn(c0, __fma_rn(x, dR, -__dmul_rn(y, dI)));
        const double nI = __dmul_rn(c0, __fma_rn(x, dI, __dmul_rn(y, dR)));
        dR = nR;
        dI = nI;
      }
      if (mm == 0) {
        const double i1 = __dmul_rn(zr, dR);
        const double cs = __fma_rn(col[0].b1R, i1, __dmul_rn(__dmul_rn(-ir2, col[0].b2R), dR));
        acc = __dadd_rn(acc, cs);
      } else {
        const double cs = __fma_rn(col[i].b1R, dR, -__dmul_rn(col[i].b1I, dI));
        acc = __dadd_rn(acc, __dmul_rn(2.0, cs));
      }
    }
  }
  return -acc;
}

__device__ __forceinline__ int ff_nterms(int P) { return (P + 1) * (P + 2) / 2 - 1; }

struct FFQuery {
  int32_t s;   // slot
  bool live;
  double px, py, pz, qa, qb, qc;
};

__device__ __forceinline__ FFQuery ff_query_at(int32_t t, int32_t m,
                                               const int32_t* __restrict__ order,
                                               const int32_t* __restrict__ active,
                                               const double* __restrict__ pos, const Frame& f) {
  FFQuery Q;
  Q.live = t < m;
  Q.s = Q.live ? (order ? order[t] : t) : 0;
  const int32_t q = Q.live ? (active ? active[Q.s] : Q.s) : 0;
  Q.px = Q.live ? pos[3 * (int64_t)q] : 0.0;
  Q.py = Q.live ? pos[3 * (int64_t)q + 1] : 0.0;
  Q.pz = Q.live ? pos[3 * (int64_t)q + 2] : 0.0;
  frame_q(f, Q.px, Q.py, Q.pz, Q.qa, Q.qb, Q.qc);
  return Q;
}

// one query per thread, or per warp (kWarp: small rounds)
template <bool kWarp>
__device__ __forceinline__ FFQuery ff_query(int32_t m, const int32_t* __restrict__ order,
                                            const int32_t* __restrict__ active,
                                            const double* __restrict__ pos, const Frame& f) {
  const int32_t t = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) / (kWarp ? 32 : 1));
  return ff_query_at(t, m, order, active, pos, f);
}

struct FFList {
  const int32_t* ent;
  int32_t b, n;
  int64_t leaf;   // -1: none (outside the cube, or no local expansions)
};

struct FFLocal {
  const int32_t* loff = nullptr;  // null: no local expansions this round
  const int32_t* lent = nullptr;
  const double2* leafL = nullptr;
  int n = 0;                      // leaves per axis
  int64_t n_leaf = 0;
  double x0 = 0, y0 = 0, z0 = 0, h = 0, side = 0;
};

__device__ __forceinline__ FFList ff_list(const FFLocal& F, int32_t C, const FFQuery& Q) {
  FFList l{nullptr, 0, C, -1};
  if (!F.loff || !Q.live) return l;
  const double ux = (Q.px - F.x0) / F.side, uy = (Q.py - F.y0) / F.side,
               uz = (Q.pz - F.z0) / F.side;
  int64_t li = F.n_leaf;  // the outside list: every entry
  if (ux >= 0.0 && ux < 1.0 && uy >= 0.0 && uy < 1.0 && uz >= 0.0 && uz < 1.0) {
    const int64_t ix = min((int64_t)(ux * F.n), (int64_t)F.n - 1);
    const int64_t iy = min((int64_t)(uy * F.n), (int64_t)F.n - 1);
    const int64_t iz = min((int64_t)(uz * F.n), (int64_t)F.n - 1);
    li = (ix * F.n + iy) * F.n + iz;
    l.leaf = li;
  }
  l.ent = F.lent;
  l.b = __ldg(F.loff + li);
  l.n = __ldg(F.loff + li + 1) - l.b;
  return l;
}

__device__ __forceinline__ int32_t ff_entry(const FFList& l, int j) {
  return j < l.n ? (l.ent ? __ldg(l.ent + l.b + j) : j) : -1;
}

constexpr int kFFBlock = 128;
#ifndef GWN_FF_WARP_QUERIES
#define GWN_FF_WARP_QUERIES 4736
#endif
constexpr int kFFWarpRoundThreads = GWN_FF_WARP_QUERIES * 32;  // rounds up to this many queries: a warp each

// warp-aggregated atomicAdd of 1 per lane on counter[c] (lanes of `mask`
// with equal c share one atomic); returns the lane's slot
__device__ __forceinline__ unsigned ff_append(unsigned mask, int32_t c, unsigned* counter) {
  const int lane = threadIdx.x & 31;
  const unsigned grp = __match_any_sync(mask, c);
  const int leader = __ffs(grp) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(counter + c, (unsigned)__popc(grp));
  base = __shfl_sync(grp, base, leader);
  return base + (unsigned)__popc(grp & ((1u << lane) - 1u));
}

// far-pair value: the entry's expansion at the lane's order (the warp runs
// to its largest order P), plus a sliver's exact chord term (the edge's fan
// sum = Omega(edge + chord back) + the chord's forward fan term, K4's shifted
// form in the ray frame; den > 0: the half-line misses the sliver's sphere)
// the lowest order level whose truncation bound holds at the pair's distance
__device__ __forceinline__ int ff_level_of(const FFRound& R, const FFQuery& Q, int32_t c,
                                           double& x, double& y, double& z) {
  x = __dsub_rn(Q.px, __ldg(R.gw + 3 * c));
  y = __dsub_rn(Q.py, __ldg(R.gw + 3 * c + 1));
  z = __dsub_rn(Q.pz, __ldg(R.gw + 3 * c + 2));
  const double R2 = __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
  const double* lv = R.lv + (int64_t)kFFLevels * c;
  int lvl = kFFLevels - 1;
#pragma unroll
  for (int l = 0; l < kFFLevels - 1; ++l)
    if (lvl == kFFLevels - 1 && R2 > __ldg(lv + l)) lvl = l;
  return lvl;
}

__device__ __forceinline__ int ff_level(const FFRound& R, const FFQuery& Q, int32_t c) {
  double x, y, z;
  return ff_level_of(R, Q, c, x, y, z);
}

__device__ __forceinline__ double ff_chord_term(const FFRound& R, const FFQuery& Q, int32_t c) {
  const double* A = R.ffa + 6 * (int64_t)c;
  const double rax = __ldg(A) - Q.qa, ray = __ldg(A + 1) - Q.qb, raz = __ldg(A + 2) - Q.qc;
  const double rbx = __ldg(A + 3) - Q.qa, rby = __ldg(A + 4) - Q.qb, rbz = __ldg(A + 5) - Q.qc;
  const double ia = 1.0 / sqrt(rax * rax + ray * ray + raz * raz);
  const double ib = 1.0 / sqrt(rbx * rbx + rby * rby + rbz * rbz);
  const double uax = rax * ia, uay = ray * ia, uaz = fma(raz, ia, -1.0);
  const double ubx = rbx * ib, uby = rby * ib, ubz = fma(rbz, ib, -1.0);
  const double num = uay * ubx - uax * uby;
  const double den = uax * ubx + uay * uby + uaz * ubz;
  return 2.0 * atan2(num, den);
}

__device__ __forceinline__ double ff_pair_value(const FFRound& R, const FFQuery& Q, int32_t c,
                                                bool far, int wind, unsigned long long& terms) {
  if (!far) return 0.0;
  double x, y, z;
  const int pl = ff_order(ff_level_of(R, Q, c, x, y, z));
  // four columns at a time at the lane's own order (bit-identical to the
  // one-column evaluation at any warp order, see ff_eval_own; its dependent
  // chain is 4x shorter, which is what bounds a warp-per-query round)
  double v = ff_eval_own(x, y, z, R.D + (int64_t)c * kFFTerms, pl);
  terms += (unsigned long long)ff_nterms(pl);
  if (__ldg(R.chord + c) >= 0) v = __dadd_rn(v, ff_chord_term(R, Q, c));
  if (wind) v = __dadd_rn(v, kShadowJump * (double)wind);
  return v;
}

__device__ __forceinline__ double ff_local(const FFLocal& F, const FFList& L, const FFQuery& Q) {
  const int64_t n = F.n, ix = L.leaf / (n * n), iy = (L.leaf / n) % n, iz = L.leaf % n;
  const double zx = F.x0 + ((double)ix + 0.5) * F.h, zy = F.y0 + ((double)iy + 0.5) * F.h,
               zz = F.z0 + ((double)iz + 0.5) * F.h;
  return fmm_l2p(Q.px - zx, Q.py - zy, Q.pz - zz, F.leafL + L.leaf * kFmmLT);
}

// Count pass: near pairs per query (qcnt) and per entry (ecnt).
// kWarp = false: a thread per query, the warp steps through its lanes' lists
// together (lanes of one leaf share the list); kWarp = true (small rounds):
// a warp per query, 32 entries at a time.
template <bool kWarp>
__global__ void __launch_bounds__(kFFBlock)
k_ff_count(int32_t m, const int32_t* __restrict__ order, const int32_t* __restrict__ active,
           const double* __restrict__ pos, Frame f, FFRound R, FFLocal F,
           unsigned* __restrict__ qcnt, unsigned* __restrict__ ecnt, unsigned* __restrict__ qfcnt,
           unsigned* __restrict__ lcnt, unsigned long long* __restrict__ counters) {
  const FFQuery Q = ff_query<kWarp>(m, order, active, pos, f);
  const FFList L = ff_list(F, R.C, Q);
  const int lane = threadIdx.x & 31;
  unsigned n = 0;
  if (kWarp) {
    for (int j0 = 0; Q.live && j0 < L.n; j0 += 32) {  // warp-uniform (one query)
      const int32_t c = ff_entry(L, j0 + lane);
      int wd;
      const bool near = c >= 0 && ff_class(R, c, Q.qa, Q.qb, Q.qc, wd) == 0;
      if (near) atomicAdd(ecnt + c, 1u);
      n += (unsigned)__popc(__ballot_sync(0xffffffffu, near));
    }
    if (Q.live && lane == 0) {
      qcnt[Q.s] = n;
      if (n) atomicAdd(&counters[CNT_NEAR], (unsigned long long)n);
    }
    return;
  }
  unsigned nf = 0;
  const int jn = (int)__reduce_max_sync(0xffffffffu, Q.live ? (unsigned)L.n : 0u);
  for (int j = 0; j < jn; ++j) {  // warp-uniform loop
    const int32_t c = Q.live ? ff_entry(L, j) : -1;
    int wd;
    const bool far = c >= 0 && ff_class(R, c, Q.qa, Q.qb, Q.qc, wd) > 0;
    const bool near = c >= 0 && !far;
    n += near ? 1u : 0u;
    const unsigned b = __ballot_sync(0xffffffffu, near);
    if (near) ff_append(b, c, ecnt);
    const unsigned fb = __ballot_sync(0xffffffffu, far);
    if (far) {  // bucket (order level, entry): a warp of the eval shares both
      ++nf;
      ff_append(fb, ff_level(R, Q, c) * R.C + c, lcnt);
    }
  }
  if (Q.live) {
    qcnt[Q.s] = n;
    qfcnt[Q.s] = nf;
  }
  unsigned long long tot = n;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
  if (lane == 0 && tot) atomicAdd(&counters[CNT_NEAR], tot);
}

// Fill pass: the far row (local expansion + far pairs, added in list order)
// and the near-pair records (slot, ordinal) of every entry.  Both variants
// give a query the same bits: its pair values are computed per lane at the
// lane's own order and folded into one sum in list order.
template <bool kWarp>
__global__ void __launch_bounds__(kFFBlock)
k_ff_fill(int32_t m, const int32_t* __restrict__ order, const int32_t* __restrict__ active,
          const double* __restrict__ pos, Frame f, FFRound R, FFLocal F,
          const unsigned long long* __restrict__ eoff, unsigned* __restrict__ efill,
          int2* __restrict__ recs, const unsigned long long* __restrict__ loffs,
          unsigned* __restrict__ lfill, int2* __restrict__ frecs, int32_t* __restrict__ fent,
          double* __restrict__ fpos, double* __restrict__ row_far,
          unsigned long long* __restrict__ counters) {
  const FFQuery Q = ff_query<kWarp>(m, order, active, pos, f);
  const FFList L = ff_list(F, R.C, Q);
  const int lane = threadIdx.x & 31;
  double om = 0.0;
  unsigned long long nfar = 0, terms = 0, nloc = 0, nsh = 0;
  if (L.leaf >= 0) {  // the leaf's local expansion: every cycle its ancestors took
    om = ff_local(F, L, Q);
    nloc = (!kWarp || lane == 0) ? 1 : 0;
  }
  if (kWarp) {
    int k = 0;
    for (int j0 = 0; Q.live && j0 < L.n; j0 += 32) {  // warp-uniform (one query)
      const int32_t c = ff_entry(L, j0 + lane);
      int wd = 0;
      const int cls = c >= 0 ? ff_class(R, c, Q.qa, Q.qb, Q.qc, wd) : 0;
      const bool far = cls > 0;
      const bool near = c >= 0 && !far;
      const unsigned nb = __ballot_sync(0xffffffffu, near);
      if (near) {
        const unsigned slot = atomicAdd(efill + c, 1u);
        recs[eoff[c] + slot] = make_int2(Q.s, k + __popc(nb & ((1u << lane) - 1u)));
      }
      k += __popc(nb);
      const double v = ff_pair_value(R, Q, c, far, wd, terms);
      const unsigned fb = __ballot_sync(0xffffffffu, far);
      nfar += far ? 1 : 0;
      nsh += cls == 2 ? 1 : 0;
      for (int i = 0; i < 32; ++i) {  // fold in list order
        const double vi = __shfl_sync(0xffffffffu, v, i);
        if ((fb >> i) & 1u) om = __dadd_rn(om, vi);
      }
    }
    if (Q.live && lane == 0) row_far[Q.s] = 0.5 * om;
  } else {
    int k = 0, kf = 0;
    const int jn = (int)__reduce_max_sync(0xffffffffu, Q.live ? (unsigned)L.n : 0u);
    for (int j = 0; j < jn; ++j) {  // warp-uniform loop
      const int32_t c = Q.live ? ff_entry(L, j) : -1;
      int wd = 0;
      const int cls = c >= 0 ? ff_class(R, c, Q.qa, Q.qb, Q.qc, wd) : 0;
      const bool far = cls > 0;
      const bool near = c >= 0 && !far;
      const unsigned b = __ballot_sync(0xffffffffu, near);
      if (near) {  // append to entry c's near-pair list
        const unsigned slot = ff_append(b, c, efill);
        recs[eoff[c] + slot] = make_int2(Q.s, k);
        ++k;
      }
      // far: a record in its order level's bucket (k_ff_far_eval evaluates
      // each bucket at one order); lanes of one leaf share c, so a warp's
      // records of one level are contiguous
      const unsigned fb = __ballot_sync(0xffffffffu, far);
      if (far) {
        nsh += cls == 2 ? 1 : 0;
        const int key = ff_level(R, Q, c) * R.C + c;
        const unsigned slot = ff_append(fb, key, lfill);
        const unsigned long long at = loffs[key] + slot;
        frecs[at] = make_int2(Q.s, kf++);
        fent[at] = c;
        // the query's position travels with the record: k_ff_far_eval reads it
        // in record order instead of gathering it through slot -> active -> pos
        // (two dependent loads ahead of every pair: 21% of its stall samples)
        fpos[3 * at] = Q.px;
        fpos[3 * at + 1] = Q.py;
        fpos[3 * at + 2] = Q.pz;
      }
    }
    // the local expansion's value; k_ff_far_sum adds the far pairs in list
    // order and halves (K4's partials are sums of atan2: Omega / 2)
    if (Q.live) row_far[Q.s] = om;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nfar += __shfl_down_sync(0xffffffffu, nfar, o);
    terms += __shfl_down_sync(0xffffffffu, terms, o);
    nloc += __shfl_down_sync(0xffffffffu, nloc, o);
    nsh += __shfl_down_sync(0xffffffffu, nsh, o);
  }
  if (lane == 0 && nsh) atomicAdd(&counters[CNT_SHADOW], nsh);
  if (lane == 0 && nfar) {
    atomicAdd(&counters[CNT_FAR], nfar);
    atomicAdd(&counters[CNT_FAR_TERMS], terms);
  }
  if (lane == 0 && nloc) atomicAdd(&counters[CNT_LOCAL], nloc);
}

// Far pairs of the per-thread path, one thread each, bucket by bucket
// (buckets = (order level, entry): a warp's lanes agree on the order and
// read the same moments): the pair's value into its query's far slots
// (ordinal kf of the query's far pairs).
__global__ void __launch_bounds__(kFFBlock)
k_ff_far_eval(unsigned long long nrec, const int2* __restrict__ frecs,
              const int32_t* __restrict__ fent, const double* __restrict__ fpos, Frame f,
              FFRound R, const unsigned long long* __restrict__ qfoff,
              double* __restrict__ fval, unsigned long long* __restrict__ counters) {
  // the block's records share one entry almost always (buckets hold
  // thousands): its moments are staged in shared memory, read as broadcasts
  __shared__ double2 sD[kFFTerms];
  __shared__ int32_t s_c[1];
  const unsigned long long r0 = (unsigned long long)blockIdx.x * blockDim.x;
  const unsigned long long r = r0 + threadIdx.x;
  const bool live = r < nrec;
  const int2 rec = live ? frecs[r] : make_int2(0, 0);
  const int32_t c = live ? fent[r] : 0;
  FFQuery Q;
  Q.live = live;
  Q.s = rec.x;
  Q.px = live ? fpos[3 * r] : 0.0;
  Q.py = live ? fpos[3 * r + 1] : 0.0;
  Q.pz = live ? fpos[3 * r + 2] : 0.0;
  if (threadIdx.x == 0) s_c[0] = fent[r0];
  __syncthreads();
  // staged only when EVERY record of the block has the first one's entry
  // (records are ordered by (level, entry): a block over several small
  // buckets can begin and end in the same entry with others in between)
  const bool staged = __syncthreads_and(!live || c == s_c[0]) != 0;
  if (staged) {
    const double2* src = R.D + (int64_t)s_c[0] * kFFTerms;
    for (int q = threadIdx.x; q < kFFTerms; q += blockDim.x) sD[q] = __ldg(src + q);
  }
  // where the value goes: loaded ahead of the evaluation, which hides it
  const unsigned long long dst = live ? qfoff[rec.x] + (unsigned long long)rec.y : 0ull;
  __syncthreads();
  frame_q(f, Q.px, Q.py, Q.pz, Q.qa, Q.qb, Q.qc);
  unsigned long long terms = 0;
  double v = 0.0;
  if (live) {
    double x, y, z;
    const int pl = ff_order(ff_level_of(R, Q, c, x, y, z));
    if (staged)  // two inlined copies: shared-memory loads here, global below
      v = ff_eval_own(x, y, z, sD, pl);
    else
      v = ff_eval_own(x, y, z, R.D + (int64_t)c * kFFTerms, pl);
    terms = (unsigned long long)ff_nterms(pl);
    if (__ldg(R.chord + c) >= 0) v = __dadd_rn(v, ff_chord_term(R, Q, c));
    int wd;  // the pair's shadow winding number (same decision as the fill pass)
    ff_class(R, c, Q.qa, Q.qb, Q.qc, wd);
    if (wd) v = __dadd_rn(v, kShadowJump * (double)wd);
  }
  if (live) fval[dst] = v;
  unsigned long long nf = live ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nf += __shfl_down_sync(0xffffffffu, nf, o);
    terms += __shfl_down_sync(0xffffffffu, terms, o);
  }
  if ((threadIdx.x & 31) == 0 && nf) {
    atomicAdd(&counters[CNT_FAR], nf);
    atomicAdd(&counters[CNT_FAR_TERMS], terms);
  }
}

// per query: local expansion value + far pairs in list order, halved
__global__ void k_ff_far_sum(int32_t m, const unsigned long long* __restrict__ qfoff,
                             const double* __restrict__ fval, double* __restrict__ row) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  double a = row[s];
  for (unsigned long long p = qfoff[s]; p < qfoff[s + 1]; ++p) a = __dadd_rn(a, fval[p]);
  row[s] = 0.5 * a;
}

// tiles of kBlockQ * kNearQPT near pairs per entry
__global__ void k_ff_tiles(int32_t C, const unsigned* __restrict__ ecnt, int tp,
                           unsigned* __restrict__ tcnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) tcnt[c] = (ecnt[c] + tp - 1) / tp;
}

template <int QPT>
__global__ void __launch_bounds__(kBlockQ, kNearMinBlocks)
k_ff_near(int32_t C, const unsigned long long* __restrict__ toff,
          const unsigned long long* __restrict__ eoff, const int32_t* __restrict__ ent_eoff,
          const int2* __restrict__ recs, const unsigned long long* __restrict__ qoff,
          const int32_t* __restrict__ active, const double* __restrict__ pos,
          const double* __restrict__ vproj, int64_t V, int S, const double* __restrict__ band_h,
          Frame f, DevParams prm, double* __restrict__ slot_ang,
          int32_t* __restrict__ flag_acc, unsigned long long* __restrict__ counters) {
  // entry of this tile: the last c with toff[c] <= tile (block-uniform search)
  const unsigned long long tile = blockIdx.x;
  int lo = 0, hi = C;  // toff[lo] <= tile < toff[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(toff + mid) <= tile) lo = mid; else hi = mid;
  }
  const int c = lo;
  const unsigned long long p_beg = eoff[c] + (tile - toff[c]) * (unsigned long long)(kBlockQ * QPT);
  const unsigned long long p_end = min(eoff[c + 1], p_beg + (unsigned long long)(kBlockQ * QPT));
  const int64_t E0 = ent_eoff[c], E1 = ent_eoff[c + 1];
  const int ept = kTileV / S;
  __shared__ double sx[kTileV], sy[kTileV], sz[kTileV];
  int32_t qs[QPT], qk[QPT];
  double qa[QPT], qb[QPT], qc[QPT];
  SegState st[QPT];
  int flags[QPT], minhi[QPT], neg[QPT];
  bool live[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    const unsigned long long p = p_beg + (unsigned long long)(j * kBlockQ + threadIdx.x);
    live[j] = p < p_end;
    const int2 r = live[j] ? recs[p] : make_int2(0, 0);
    qs[j] = r.x;
    qk[j] = r.y;
    const int32_t q = live[j] ? (active ? active[r.x] : r.x) : 0;
    const double px = live[j] ? pos[3 * (int64_t)q] : 0.0;
    const double py = live[j] ? pos[3 * (int64_t)q + 1] : 0.0;
    const double pz = live[j] ? pos[3 * (int64_t)q + 2] : 0.0;
    qa[j] = px * f.e1[0] + py * f.e1[1] + pz * f.e1[2];
    qb[j] = px * f.e2[0] + py * f.e2[1] + pz * f.e2[2];
    qc[j] = px * f.d[0] + py * f.d[1] + pz * f.d[2];
    st[j] = SegState{1.0, 0.0, 0};
    flags[j] = 0;
    minhi[j] = 0x7fffffff;
    neg[j] = 0;
  }
  VtxF va[QPT], vb[QPT];
  for (int64_t te = E0; te < E1; te += ept) {
    const int ne = (int)min((int64_t)ept, E1 - te);
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
    for (int e = 0; e < ne; ++e)
      edge_segments<QPT>(sx, sy, sz, e * S, S, live, qa, qb, qc, st, neg, minhi, va, vb);
    band_rewalk<QPT>(sx, sy, sz, ne, S, band_h, te, qa, qb, qc, prm.band_factor, neg, flags);
  }
  int nlive = 0;
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    if (!live[j]) continue;
    ++nlive;
    if (minhi[j] < kDegHi) flags[j] |= FLAG_DEGEN;
    slot_ang[qoff[qs[j]] + (unsigned long long)qk[j]] = seg_angle(st[j]);
    if (flags[j]) atomicOr(&flag_acc[qs[j]], flags[j]);
  }
  // exact (query, segment) pairs, one atomic per warp
  unsigned long long segs = (unsigned long long)nlive * (unsigned long long)((E1 - E0) * (S - 1));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) segs += __shfl_down_sync(0xffffffffu, segs, o);
  if ((threadIdx.x & 31) == 0 && segs) atomicAdd(&counters[CNT_SEGMENTS], segs);
}

// per query: its near angles in entry order (row 1 of the partials)
__global__ void k_ff_near_sum(int32_t m, const unsigned long long* __restrict__ qoff,
                              const double* __restrict__ slot_ang, double* __restrict__ row) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  double a = 0.0;
  for (unsigned long long p = qoff[s]; p < qoff[s + 1]; ++p) a = __dadd_rn(a, slot_ang[p]);
  row[s] = a;
}

// per host thread and device: the far-field pass buffers, grown on demand
// (gwn_eval synchronises before returning, so the next eval reuses them)
struct FFCache {
  size_t cap_q = 0, cap_c = 0, cap_p = 0, cap_tmp = 0;
  unsigned* qcnt = nullptr;              // (m+1)
  unsigned long long* qoff = nullptr;    // (m+1)
  unsigned* ecnt = nullptr;              // (C+1) counts, then fill cursors
  unsigned* efill = nullptr;             // (C+1)
  unsigned* tcnt = nullptr;              // (C+1)
  unsigned long long* eoff = nullptr;    // (C+1)
  unsigned long long* toff = nullptr;    // (C+1)
  int2* recs = nullptr;                  // (pairs)
  double* ang = nullptr;                 // (pairs)
  // far pairs of the per-thread path
  size_t cap_f = 0;
  unsigned* qfcnt = nullptr;             // (m+1)
  unsigned long long* qfoff = nullptr;   // (m+1)
  size_t cap_k = 0;
  unsigned* lcnt = nullptr;              // (kFFLevels*C + 1) bucket sizes
  unsigned* lfill = nullptr;             // (kFFLevels*C) bucket cursors
  unsigned long long* loffs = nullptr;   // (kFFLevels*C + 1)
  int2* frecs = nullptr;                 // (far pairs) (slot, ordinal)
  int32_t* fent = nullptr;               // (far pairs) entry
  double* fpos = nullptr;                // (far pairs, 3) query position of the pair
  double* fval = nullptr;                // (far pairs) values by (query, ordinal)
  void* tmp = nullptr;
  unsigned long long* h = nullptr;       // pinned: [0] pairs, [1] tiles, [2] far pairs
};
static thread_local FFCache t_ffc[64];

void release_boundary_caches(int device) {
  FFCache& c = t_ffc[device & 63];
  void* ps[] = {c.qcnt, c.qoff, c.ecnt, c.efill, c.tcnt, c.eoff, c.toff, c.recs, c.ang, c.tmp,
                c.qfcnt, c.qfoff, c.lcnt, c.lfill, c.loffs, c.frecs, c.fent, c.fval, c.fpos};
  for (void* p : ps)
    if (p) cudaFree(p);
  unsigned long long* h = c.h;
  c = FFCache();
  c.h = h;  // the pinned scalars stay
}

template <class T>
static cudaError_t ff_grow(T*& p, size_t& cap, size_t n, size_t unit, cudaStream_t st) {
  if (cap >= n) return cudaSuccess;
  if (p) cudaFreeAsync(p, st);
  p = nullptr;
  cap = 0;
  const size_t want = n + n / 4 + 1024;
  cudaError_t e = cudaMallocAsync((void**)&p, want * unit, st);
  if (e == cudaSuccess) cap = want;
  return e;
}

static cudaError_t launch_boundary_ff(const gwn_scene* sc, const Round& rd, int32_t m,
                                      const int32_t* active, const double* pos, double* bpart,
                                      int32_t* flags, unsigned long long* counters,
                                      cudaStream_t st, const int32_t* order, cudaEvent_t* evb) {
  FFCache& c = t_ffc[sc->device & 63];
  const int32_t C = sc->ff_n;
  const int nkey = kFFLevels * C;  // far-pair buckets (order level, entry)
  const int64_t V = sc->n_edges * sc->S;
  const int tp = kBlockQ * kNearQPT;
  cudaError_t e = cudaSuccess;
#define FC(x)                              \
  do {                                     \
    if ((e = (x)) != cudaSuccess) return e; \
  } while (0)
  if (!c.h) FC(cudaHostAlloc((void**)&c.h, 4 * sizeof(unsigned long long), cudaHostAllocPortable));
  {
    size_t capq = c.cap_q;
    FC(ff_grow(c.qcnt, capq, (size_t)m + 1, sizeof(unsigned), st));
    capq = c.cap_q;
    FC(ff_grow(c.qoff, capq, (size_t)m + 1, sizeof(unsigned long long), st));
    capq = c.cap_q;
    FC(ff_grow(c.qfcnt, capq, (size_t)m + 1, sizeof(unsigned), st));
    capq = c.cap_q;
    FC(ff_grow(c.qfoff, capq, (size_t)m + 1, sizeof(unsigned long long), st));
    c.cap_q = capq;
    size_t capk = c.cap_k;
    FC(ff_grow(c.lcnt, capk, (size_t)nkey + 1, sizeof(unsigned), st));
    capk = c.cap_k;
    FC(ff_grow(c.lfill, capk, (size_t)nkey + 1, sizeof(unsigned), st));
    capk = c.cap_k;
    FC(ff_grow(c.loffs, capk, (size_t)nkey + 1, sizeof(unsigned long long), st));
    c.cap_k = capk;
    size_t capc = c.cap_c;
    FC(ff_grow(c.ecnt, capc, (size_t)C + 1, sizeof(unsigned), st));
    capc = c.cap_c;
    FC(ff_grow(c.efill, capc, (size_t)C + 1, sizeof(unsigned), st));
    capc = c.cap_c;
    FC(ff_grow(c.tcnt, capc, (size_t)C + 1, sizeof(unsigned), st));
    capc = c.cap_c;
    FC(ff_grow(c.eoff, capc, (size_t)C + 1, sizeof(unsigned long long), st));
    capc = c.cap_c;
    FC(ff_grow(c.toff, capc, (size_t)C + 1, sizeof(unsigned long long), st));
    c.cap_c = capc;
  }
  size_t tb1 = 0, tb2 = 0, tb3 = 0;
  FC(cub::DeviceScan::ExclusiveSum(nullptr, tb1, c.qcnt, c.qoff, m + 1, st));
  FC(cub::DeviceScan::ExclusiveSum(nullptr, tb2, c.ecnt, c.eoff, C + 1, st));
  FC(cub::DeviceScan::ExclusiveSum(nullptr, tb3, c.lcnt, c.loffs, nkey + 1, st));
  FC(ff_grow(c.tmp, c.cap_tmp, std::max(std::max(tb1, tb2), tb3), 1, st));
  const FFRound R{C,        rd.ffg,   sc->ff_r, sc->ff_lv, sc->ff_g,
                  reinterpret_cast<const double2*>(sc->ff_D), sc->ff_chord, rd.ffa,
                  rd.ffw,   rd.ffwg};
  FFLocal F;
  if (rd.fmm) {  // round 0 of a scene with local expansions (gwn_fmm.cu)
    F.loff = rd.fmm->loff;
    F.lent = rd.fmm->lent;
    F.leafL = rd.fmm->leafL;
    F.n = 1 << rd.fmm->L;
    F.n_leaf = rd.fmm->n_leaf;
    F.x0 = sc->fmm_x0[0];
    F.y0 = sc->fmm_x0[1];
    F.z0 = sc->fmm_x0[2];
    F.side = sc->fmm_side;
    F.h = sc->fmm_side / (double)F.n;
  }
  FC(cudaMemsetAsync(c.ecnt, 0, sizeof(unsigned) * (C + 1), st));
  FC(cudaMemsetAsync(c.efill, 0, sizeof(unsigned) * (C + 1), st));
  FC(cudaMemsetAsync(c.qcnt + m, 0, sizeof(unsigned), st));
  FC(cudaMemsetAsync(c.qfcnt + m, 0, sizeof(unsigned), st));
  FC(cudaMemsetAsync(c.lcnt, 0, sizeof(unsigned) * (nkey + 1), st));
  // small rounds (re-shoots): a warp per query, so the few queries' pairs
  // spread over the GPU instead of serialising in one block; it evaluates its
  // far pairs in place (no far-pair lists)
  const bool per_warp = (int64_t)m * 32 <= (int64_t)kFFWarpRoundThreads;
  const unsigned g = per_warp ? (unsigned)(((int64_t)m * 32 + kFFBlock - 1) / kFFBlock)
                              : (unsigned)((m + kFFBlock - 1) / kFFBlock);
  if (per_warp)
    k_ff_count<true><<<g, kFFBlock, 0, st>>>(m, order, active, pos, rd.f, R, F, c.qcnt, c.ecnt,
                                             c.qfcnt, c.lcnt, counters);
  else
    k_ff_count<false><<<g, kFFBlock, 0, st>>>(m, order, active, pos, rd.f, R, F, c.qcnt,
                                              c.ecnt, c.qfcnt, c.lcnt, counters);
  FC(cudaGetLastError());
  FC(cub::DeviceScan::ExclusiveSum(c.tmp, tb1, c.qcnt, c.qoff, m + 1, st));
  if (!per_warp) {
    FC(cub::DeviceScan::ExclusiveSum(c.tmp, tb1, c.qfcnt, c.qfoff, m + 1, st));
    FC(cub::DeviceScan::ExclusiveSum(c.tmp, tb3, c.lcnt, c.loffs, nkey + 1, st));
    FC(cudaMemsetAsync(c.lfill, 0, sizeof(unsigned) * nkey, st));
    FC(cudaMemcpyAsync(c.h + 2, c.qfoff + m, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       st));
  }
  FC(cub::DeviceScan::ExclusiveSum(c.tmp, tb2, c.ecnt, c.eoff, C + 1, st));
  k_ff_tiles<<<(C + 255) / 256, 256, 0, st>>>(C + 1, c.ecnt, tp, c.tcnt);
  FC(cudaGetLastError());
  FC(cub::DeviceScan::ExclusiveSum(c.tmp, tb2, c.tcnt, c.toff, C + 1, st));
  // near-pair and tile totals to the host: they size the pair buffers and
  // the exact kernel's grid (one round trip per round and chunk)
  FC(cudaMemcpyAsync(c.h, c.qoff + m, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  FC(cudaMemcpyAsync(c.h + 1, c.toff + C, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     st));
  FC(cudaStreamSynchronize(st));
  const unsigned long long pairs = c.h[0], tiles = c.h[1], fpairs = per_warp ? 0 : c.h[2];
  {
    size_t capp = c.cap_p;
    FC(ff_grow(c.recs, capp, (size_t)pairs + 1, sizeof(int2), st));
    capp = c.cap_p;
    FC(ff_grow(c.ang, capp, (size_t)pairs + 1, sizeof(double), st));
    c.cap_p = capp;
    size_t capf = c.cap_f;
    FC(ff_grow(c.frecs, capf, (size_t)fpairs + 1, sizeof(int2), st));
    capf = c.cap_f;
    FC(ff_grow(c.fent, capf, (size_t)fpairs + 1, sizeof(int32_t), st));
    capf = c.cap_f;
    FC(ff_grow(c.fval, capf, (size_t)fpairs + 1, sizeof(double), st));
    capf = c.cap_f;
    FC(ff_grow(c.fpos, capf, (size_t)fpairs + 1, 3 * sizeof(double), st));
    c.cap_f = capf;
  }
  if (evb) FC(cudaEventRecord(evb[0], st));
  if (per_warp)
    k_ff_fill<true><<<g, kFFBlock, 0, st>>>(m, order, active, pos, rd.f, R, F, c.eoff, c.efill,
                                            c.recs, c.loffs, c.lfill, c.frecs, c.fent, c.fpos,
                                            bpart, counters);
  else
    k_ff_fill<false><<<g, kFFBlock, 0, st>>>(m, order, active, pos, rd.f, R, F, c.eoff, c.efill,
                                             c.recs, c.loffs, c.lfill, c.frecs, c.fent, c.fpos,
                                             bpart, counters);
  FC(cudaGetLastError());
  if (!per_warp) {
    if (fpairs > 0) {
      k_ff_far_eval<<<(unsigned)((fpairs + kFFBlock - 1) / kFFBlock), kFFBlock, 0, st>>>(
          fpairs, c.frecs, c.fent, c.fpos, rd.f, R, c.qfoff, c.fval, counters);
      FC(cudaGetLastError());
    }
    k_ff_far_sum<<<(m + 255) / 256, 256, 0, st>>>(m, c.qfoff, c.fval, bpart);
    FC(cudaGetLastError());
  }
  if (evb) FC(cudaEventRecord(evb[1], st));
  if (tiles > 0) {
    k_ff_near<kNearQPT><<<(unsigned)tiles, kBlockQ, 0, st>>>(
        C, c.toff, c.eoff, sc->ff_eoff, c.recs, c.qoff, active, pos, rd.vproj, V, sc->S,
        sc->band_h, rd.f, sc->dprm, c.ang, flags, counters);
    FC(cudaGetLastError());
  }
  if (evb) FC(cudaEventRecord(evb[2], st));
  k_ff_near_sum<<<(m + 255) / 256, 256, 0, st>>>(m, c.qoff, c.ang, bpart + m);
  FC(cudaGetLastError());
#undef FC
  return cudaSuccess;
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

// Shadow winding grid of closed expanded entry c (one block): kWG x kWG
// cells over the square around the disk of the cycle's sphere projected
// along d (X, Y of the round frame).  A cell holds the winding number of the
// cycle's projection around the cell centre, or kWDirty when some vertex's
// projection lies within del = 2.02 Lmax of the cell (Lmax: the entry's
// longest 3-D segment).
// Why that makes a clean cell exact: a segment (a, b) of the fan sum has
// den = (a^ - d).(b^ - d) (a^ = the unit vector from the query to a); den < 0
// forces |a^ - d| < |a^ - b^| <= 2|a - b| / (|a - q| + |b - q|), so the
// perpendicular distance of a from the query's line is below 2|a - b|.  In
// a clean cell no segment has den < 0 (no branch flip, no band test: the
// exact kernel would raise no flag) and no projected segment passes through
// the cell (its end points would lie within Lmax of it), so the cell's
// winding number is the query's.  The fan sum then equals Omega/2 of the
// cycle's fan surface plus 2 pi times that winding number (the forward
// half-line crosses the fan surface wind times, all at t > 0).
__global__ void __launch_bounds__(256)
k_ff_wind(int32_t C, const int32_t* __restrict__ ent_eoff, const int32_t* __restrict__ chord,
          const double* __restrict__ r2, const double* __restrict__ g3,
          const double* __restrict__ vproj, int64_t V, int S, int8_t* __restrict__ wg,
          double* __restrict__ wgeo) {
  const int c = blockIdx.x;
  const int t = threadIdx.x;
  __shared__ int cr[kWG + 1], dr[kWG + 1];
  __shared__ double s_red[8];
  const double rmin2 = r2[2 * c], line2 = r2[2 * c + 1];
  const double line = sqrt(line2);
  const double x0 = g3[3 * c] - line, y0 = g3[3 * c + 1] - line;
  const double h = 2.0 * line / kWG, ih = kWG / (2.0 * line);
  int8_t* out = wg + (int64_t)c * kWG * kWG;
  if (t == 0) {
    wgeo[3 * c] = x0;
    wgeo[3 * c + 1] = y0;
    wgeo[3 * c + 2] = ih;
  }
  // closed expanded cycles only (slivers keep their chord term exact)
  if (!(chord[c] < 0 && rmin2 < INFINITY && rmin2 > line2 && line > 0.0)) {
    for (int k = t; k < kWG * kWG; k += blockDim.x) out[k] = (int8_t)kWDirty;
    return;
  }
  const int64_t v0 = (int64_t)ent_eoff[c] * S, v1 = (int64_t)ent_eoff[c + 1] * S;
  double lm = 0.0;
  for (int64_t k = v0 + t; k < v1; k += blockDim.x) {
    if ((k - v0) % S == S - 1) continue;  // an edge's last sample starts no segment
    const double ex = vproj[k + 1] - vproj[k], ey = vproj[V + k + 1] - vproj[V + k],
                 ez = vproj[2 * V + k + 1] - vproj[2 * V + k];
    lm = fmax(lm, ex * ex + ey * ey + ez * ez);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
  if ((t & 31) == 0) s_red[t >> 5] = lm;
  __syncthreads();
  lm = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) lm = fmax(lm, s_red[w]);
  // 1% over the bound, plus the rounding of the coordinates
  const double del = 2.02 * sqrt(lm) + 1e-6 * h + 1e-12 * (fabs(x0) + fabs(y0) + line);
  for (int row = 0; row < kWG; ++row) {
    const double yc = y0 + (row + 0.5) * h;
    for (int k = t; k <= kWG; k += blockDim.x) {
      cr[k] = 0;
      dr[k] = 0;
    }
    __syncthreads();
    for (int64_t k = v0 + t; k < v1; k += blockDim.x) {
      const double ax = vproj[k], ay = vproj[V + k];
      if (fabs(ay - yc) <= del + 0.5 * h) {  // cells within del of the vertex
        const double lo = (ax - del - x0) * ih, hi = (ax + del - x0) * ih;
        if (hi >= 0.0 && lo < (double)kWG) {
          const int ka = lo < 0.0 ? 0 : (int)lo;
          const int kb = hi >= (double)kWG ? kWG - 1 : (int)hi;
          atomicAdd(&dr[ka], 1);
          atomicAdd(&dr[kb + 1], -1);
        }
      }
      if ((k - v0) % S == S - 1) continue;
      const double by = vproj[V + k + 1];
      if ((ay <= yc) != (by <= yc)) {  // the segment crosses the row's centre line
        const double bx = vproj[k + 1];
        const double xc = ax + (yc - ay) * (bx - ax) / (by - ay);
        // cells whose centre lies left of the crossing count it (+x ray)
        const double f = (xc - x0) * ih - 0.5;
        const int kc = f <= 0.0 ? 0 : (f >= (double)kWG ? kWG : (int)ceil(f));
        const int dir = by > ay ? 1 : -1;
        if (kc > 0) {
          atomicAdd(&cr[0], dir);
          atomicAdd(&cr[kc], -dir);
        }
      }
    }
    __syncthreads();
    if (t < 32) {  // prefix sums: lane t owns cells 4t .. 4t+3
      int a[4], b[4], sa = 0, sb = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        sa += cr[4 * t + i];
        sb += dr[4 * t + i];
        a[i] = sa;
        b[i] = sb;
      }
      int pa = sa, pb = sb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, pa, o), yb = __shfl_up_sync(0xffffffffu, pb, o);
        if (t >= o) {
          pa += ya;
          pb += yb;
        }
      }
      pa -= sa;
      pb -= sb;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int wv = pa + a[i], dv = pb + b[i];
        out[row * kWG + 4 * t + i] =
            (int8_t)(dv > 0 || wv <= kWDirty || wv > 127 ? kWDirty : wv);
      }
    }
    __syncthreads();
  }
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
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (sc->ff_n > 0) {
    if ((e = cudaMalloc(&rd.ffw, (size_t)sc->ff_n * kWG * kWG)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&rd.ffwg, sizeof(double) * 3 * (size_t)sc->ff_n)) != cudaSuccess)
      return e;
    k_ff_wind<<<(unsigned)sc->ff_n, 256, 0, st>>>(sc->ff_n, sc->ff_eoff, sc->ff_chord, sc->ff_r,
                                                  rd.ffg, rd.vproj, V, sc->S, rd.ffw, rd.ffwg);
  }
  return cudaGetLastError();
}



// Edge chunks of the boundary sum.  Fixed per scene (not per batch) so the
// chunk partials -- added in chunk order by K5 -- make w bit-identical for any
// batching, chunking or sharding; enough chunks that small batches still fill
// the GPU.  Far-field scenes: two rows (far sum, near sum).
int boundary_chunks(const gwn_scene* sc, int32_t m) {
  (void)m;
  if (sc->n_edges <= 0) return 1;
  if (sc->ff_n > 0) return 2;
  return (int)std::min<int64_t>(sc->n_edges, 64);
}

// nchunk partial rows.  `order` (nullable) is the far-field passes' thread ->
// slot map (launch_ff_order); evb (nullable): 3 events recorded before the
// far pass, after it and after the exact near kernel (timing mode).
cudaError_t launch_boundary(const gwn_scene* sc, const Round& rd, int32_t m,
                            const int32_t* active, const double* pos, double* bpart, int nchunk,
                            int32_t* flags, unsigned long long* counters, cudaStream_t st,
                            const int32_t* order, cudaEvent_t* evb) {
  if (m <= 0) return cudaSuccess;
  int64_t V = sc->n_edges * sc->S;
  if (V == 0) return cudaMemsetAsync(bpart, 0, sizeof(double) * m, st);
  if (sc->ff_n > 0 && rd.ffg)
    return launch_boundary_ff(sc, rd, m, active, pos, bpart, flags, counters, st, order, evb);
  dim3 grid((m + kBlockQ * kQPT - 1) / (kBlockQ * kQPT), nchunk);
  if (sc->S <= kTileV) {
    k_boundary_e<kQPT><<<grid, kBlockQ, 0, st>>>(m, active, pos, rd.vproj, V, sc->S, sc->n_edges,
                                                 sc->band_h, rd.f, sc->dprm, bpart, flags,
                                                 counters);
  } else {
    k_boundary<kQPT><<<grid, kBlockQ, 0, st>>>(m, active, pos, rd.vproj, V, sc->S, sc->n_edges,
                                               sc->band_h, rd.f, sc->dprm, bpart, flags,
                                               counters);
  }
  return cudaGetLastError();
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
