// gwn_bvh.cu -- K1: per-direction patch projection and on-device 2-D LBVH.
//
// Every query of round r casts its ray along the same direction d_r, so the
// ray-patch cull is a 2-D point query in the plane normal to d_r: a ray from
// p can hit a piece of patch only if (p.e1, p.e2) lies in the piece's
// projected control box and the piece extends past p along d_r.  Per round we
// (1) project the control nets into the ray frame (replacing the
// per-(ray,patch) Aabb work of surfaces.py:636-639 / geometry.py:198-219),
// (2) cut every patch into adaptive leaf sub-patches carrying the
// query-independent Krawczyk data, and (3) build a Karras LBVH
// over the leaves' projected boxes: 30-bit Morton codes, CUB radix sort, one
// thread per internal node, bottom-up refit with atomic arrival counters.
#include <cub/cub.cuh>

#include <algorithm>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gwn_patch.cuh"

namespace gwn {

// cubic Bernstein coefficients -> power basis (p(t) = c0 + c1 t + c2 t^2 + c3 t^3)
__device__ __forceinline__ void bern_to_pow(double& p0, double& p1, double& p2, double& p3) {
  const double c1 = 3.0 * (p1 - p0);
  const double c2 = 3.0 * (p0 - 2.0 * p1 + p2);
  const double c3 = (p3 - p0) + 3.0 * (p1 - p2);
  p1 = c1;
  p2 = c2;
  p3 = c3;
}

// Projected control nets of every patch in the round's frame (Bernstein, K1
// and the fallback) and the same nets in the tensor power basis, index
// 4*i+j = coefficient of u^i v^j (K3 Newton evaluates them by Horner).
__global__ void k_project(const double* __restrict__ ctrl, int64_t P, Frame f,
                          double* __restrict__ proj, double* __restrict__ powc) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double* X = ctrl + 48 * p;
  double* out = proj + 48 * p;
  double net[48];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    double x = X[3 * k], y = X[3 * k + 1], z = X[3 * k + 2];
    net[k] = x * f.e1[0] + y * f.e1[1] + z * f.e1[2];
    net[16 + k] = x * f.e2[0] + y * f.e2[1] + z * f.e2[2];
    net[32 + k] = x * f.d[0] + y * f.d[1] + z * f.d[2];
  }
#pragma unroll
  for (int k = 0; k < 48; ++k) out[k] = net[k];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double* N = net + 16 * c;
#pragma unroll
    for (int i = 0; i < 4; ++i) bern_to_pow(N[4 * i], N[4 * i + 1], N[4 * i + 2], N[4 * i + 3]);
#pragma unroll
    for (int j = 0; j < 4; ++j) bern_to_pow(N[j], N[4 + j], N[8 + j], N[12 + j]);
  }
  double* pw = powc + 48 * p;
#pragma unroll
  for (int k = 0; k < 48; ++k) pw[k] = net[k];
}

// Adaptive leaf sub-patches of every patch for this direction: depth-first
// subdivision (u/v alternating, as in K3) until the Krawczyk radii over the
// leaf box expanded by kLeafM on each side are below kLeafRmax (every root in
// the leaf then certifies from the precomputed data alone), or kLeafMaxLevel.
// kFill = false: count leaves per patch; true: write LeafRec, the leaf's
// control-box (cull primitive) and its Morton key.
// leaf depth cap
static int leaf_max_level() { return kLeafMaxLevel < kLeafLevelCap ? kLeafMaxLevel : kLeafLevelCap; }

// Conservative box expansion of patch P48 (rounding + the 1e-9 parametric
// acceptance band of surfaces.py:668: roots just outside the domain).
__device__ __forceinline__ double patch_eps(const double* __restrict__ P48) {
  double mag = 0.0, alo = INFINITY, ahi = -INFINITY, blo = INFINITY, bhi = -INFINITY;
  for (int k = 0; k < 16; ++k) {
    const double A = P48[k], B = P48[16 + k], C = P48[32 + k];
    mag = fmax(mag, fmax(fabs(A), fmax(fabs(B), fabs(C))));
    alo = fmin(alo, A); ahi = fmax(ahi, A); blo = fmin(blo, B); bhi = fmax(bhi, B);
  }
  return 1e-12 * (1.0 + mag) + 3e-9 * fmax(ahi - alo, bhi - blo);
}

// Krawczyk data of the piece `code` over its box expanded by kLeafM.
__device__ __forceinline__ KrawPre piece_kraw(const double* __restrict__ P48, uint64_t code) {
  const int L = code_level(code);
  const double wu = code_wu(L), wv = code_wv(L);
  const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
  double a[16], b[16];
  for (int k = 0; k < 16; ++k) {
    a[k] = P48[k];
    b[k] = P48[16 + k];
  }
  extract_net(a, u0 - kLeafM * wu, u0 + (1.0 + kLeafM) * wu, v0 - kLeafM * wv,
              v0 + (1.0 + kLeafM) * wv);
  extract_net(b, u0 - kLeafM * wu, u0 + (1.0 + kLeafM) * wu, v0 - kLeafM * wv,
              v0 + (1.0 + kLeafM) * wv);
  return kraw_pre(a, b);
}

__device__ __forceinline__ bool kraw_certifies(const KrawPre& kp) {
  return kp.ok && kp.R0 < kLeafRmax && kp.R1 < kLeafRmax;
}

// Leaf record (Krawczyk data, separating axes) and cull box (a lo/hi, b lo/hi,
// c max) of the piece `code` of patch p.
__device__ void make_leaf(const double* __restrict__ P48, int32_t p, uint64_t code,
                          const KrawPre& kp, double eps, LeafRec& r, double box[5]) {
  const int L = code_level(code);
  const double wu = code_wu(L), wv = code_wv(L);
  const double u0 = (double)code_iu(code) * wu, v0 = (double)code_iv(code) * wv;
  r.Ga = kp.Ga; r.Gb = kp.Gb;
  r.Y00 = kp.Y00; r.Y01 = kp.Y01; r.Y10 = kp.Y10; r.Y11 = kp.Y11;
  r.R0 = kp.R0; r.R1 = kp.R1;
  r.code = code;
  r.patch = p;
  r.ok = kp.ok;
  // the piece's own control box (convex hull of the piece over D)
  double a[16], b[16], c[16];
  for (int k = 0; k < 16; ++k) {
    a[k] = P48[k];
    b[k] = P48[16 + k];
    c[k] = P48[32 + k];
  }
  extract_net(a, u0, u0 + wu, v0, v0 + wv);
  extract_net(b, u0, u0 + wu, v0, v0 + wv);
  extract_net(c, u0, u0 + wu, v0, v0 + wv);
  double la = INFINITY, ha = -INFINITY, lb = INFINITY, hb = -INFINITY, hc = -INFINITY;
  for (int k = 0; k < 16; ++k) {
    la = fmin(la, a[k]); ha = fmax(ha, a[k]);
    lb = fmin(lb, b[k]); hb = fmax(hb, b[k]);
    hc = fmax(hc, c[k]);
  }
  hull_axes(a, b, eps + 1e-15 * (fabs(la) + fabs(ha) + fabs(lb) + fabs(hb)), r);
  box[0] = la - eps; box[1] = ha + eps; box[2] = lb - eps; box[3] = hb + eps; box[4] = hc + eps;
}

template <bool kFill>
__global__ void k_leaves(int64_t P, const double* __restrict__ proj,
                         const int64_t* __restrict__ offs, int64_t* __restrict__ counts,
                         LeafRec* __restrict__ leaves, double* __restrict__ leafbox,
                         uint32_t* __restrict__ keys, int32_t* __restrict__ ids, double amin,
                         double ainv, double bmin, double binv, int max_level) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double* P48 = proj + 48 * p;
  const double eps = patch_eps(P48);
  uint64_t stack[2 * kLeafLevelCap + 4];
  int top = 0;
  stack[top++] = 0;  // root code
  int64_t n = 0;
  const int64_t o = kFill ? offs[p] : 0;
  while (top > 0) {
    const uint64_t code = stack[--top];
    const int L = code_level(code);
    const KrawPre kp = piece_kraw(P48, code);
    const bool leaf = kraw_certifies(kp) || L >= max_level;
    if (!leaf) {
      const uint64_t iu = code_iu(code), iv = code_iv(code);
      if ((L & 1) == 0) {
        stack[top++] = make_code(L + 1, 2 * iu + 1, iv);
        stack[top++] = make_code(L + 1, 2 * iu, iv);
      } else {
        stack[top++] = make_code(L + 1, iu, 2 * iv + 1);
        stack[top++] = make_code(L + 1, iu, 2 * iv);
      }
      continue;
    }
    if (kFill) {
      const int64_t li = o + n;
      LeafRec r;
      double* lbx = leafbox + 5 * li;
      make_leaf(P48, (int32_t)p, code, kp, eps, r, lbx);
      leaves[li] = r;
      const double la = lbx[0], ha = lbx[1], lb = lbx[2], hb = lbx[3];
      const double ca = (0.5 * (la + ha) - amin) * ainv, cb = (0.5 * (lb + hb) - bmin) * binv;
      const uint32_t ia = (uint32_t)fmin(fmax(ca * 32767.0, 0.0), 32767.0);
      const uint32_t ib = (uint32_t)fmin(fmax(cb * 32767.0, 0.0), 32767.0);
      uint32_t key = 0;
      for (int bit = 0; bit < 15; ++bit)
        key |= (((ia >> bit) & 1u) << (2 * bit)) | (((ib >> bit) & 1u) << (2 * bit + 1));
      keys[li] = key;
      ids[li] = (int32_t)li;
    }
    ++n;
  }
  if (!kFill) counts[p] = n;
}

// Fold trees (query-independent, once per round).  A leaf that did not
// certify at the leaf depth cap sits on a silhouette fold of the projection.
// Its subtree is refined further, to sub_level, with the same criterion, and
// stored in depth-first preorder with skip counts: node k's subtree is
// [k, k + skip[k]), a leaf has skip 1.  Every node keeps its control box and
// separating axes (LeafRec + box), so a query near the fold walks the tree
// stacklessly with cheap exclusion tests instead of re-deriving each node's
// net (node_test), and only the uncertified sub-leaves on the fold itself
// still need the per-query subdivision fallback.
// kFill = false: count tree nodes per leaf; true: write them.
template <bool kFill>
__global__ void k_foldtree(int64_t n_leaves, const LeafRec* __restrict__ leaves,
                           const double* __restrict__ proj, int sub_level, double tree_r,
                           const int64_t* __restrict__ offs, int64_t* __restrict__ counts,
                           LeafRec* __restrict__ sub, double* __restrict__ subbox,
                           int32_t* __restrict__ subskip) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_leaves) return;
  const LeafRec L = leaves[i];
  const int32_t p = L.patch;
  int64_t n = 0;
  const int64_t o = kFill ? offs[i] : 0;
  const bool cert = L.ok && L.R0 < kLeafRmax && L.R1 < kLeafRmax;
  // certified leaves with large radii get a full two-level tree: a query whose
  // predicted root sits near the leaf border (K = t* +- R leaves the
  // certification box) is then settled by stored children, not node_test
  const bool wide = cert && fmax(L.R0, L.R1) >= tree_r;
  const int lim = wide ? code_level(L.code) + 2 : sub_level;
  if ((!cert || wide) && code_level(L.code) < lim) {
    const double* P48 = proj + 48 * (int64_t)p;
    const double eps = patch_eps(P48);
    uint64_t stack[2 * kLeafLevelCap + 4];
    int64_t open_idx[kLeafLevelCap + 2];
    int open_top[kLeafLevelCap + 2];
    int top = 0, otop = 0;
    {
      uint64_t c0, c1;
      const int lv = code_level(L.code);
      const uint64_t iu = code_iu(L.code), iv = code_iv(L.code);
      if ((lv & 1) == 0) {
        c0 = make_code(lv + 1, 2 * iu, iv);
        c1 = make_code(lv + 1, 2 * iu + 1, iv);
      } else {
        c0 = make_code(lv + 1, iu, 2 * iv);
        c1 = make_code(lv + 1, iu, 2 * iv + 1);
      }
      stack[top++] = c1;
      stack[top++] = c0;
    }
    for (;;) {
      // close the internal nodes whose subtrees are complete
      while (otop > 0 && top <= open_top[otop - 1]) {
        --otop;
        if (kFill) subskip[o + open_idx[otop]] = (int32_t)(n - open_idx[otop]);
      }
      if (top == 0) break;
      const uint64_t code = stack[--top];
      const int lv = code_level(code);
      const KrawPre kp = piece_kraw(P48, code);
      // fold trees: a certified node still splits while its radii are wide
      // (so border queries settle in stored nodes), to the depth cap
      const bool leaf = wide ? lv >= lim
                             : ((kraw_certifies(kp) && fmax(kp.R0, kp.R1) < tree_r) || lv >= lim);
      if (kFill) {
        LeafRec r;
        make_leaf(P48, p, code, kp, eps, r, subbox + 5 * (o + n));
        sub[o + n] = r;
        if (leaf) subskip[o + n] = 1;
      }
      if (!leaf) {
        open_idx[otop] = n;
        open_top[otop] = top;
        ++otop;
        const uint64_t iu = code_iu(code), iv = code_iv(code);
        if ((lv & 1) == 0) {
          stack[top++] = make_code(lv + 1, 2 * iu + 1, iv);
          stack[top++] = make_code(lv + 1, 2 * iu, iv);
        } else {
          stack[top++] = make_code(lv + 1, iu, 2 * iv + 1);
          stack[top++] = make_code(lv + 1, iu, 2 * iv);
        }
      }
      ++n;
    }
  }
  if (!kFill) counts[i] = n;
}

__device__ __forceinline__ int lbvh_delta(const uint32_t* keys, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  uint32_t a = keys[i], b = keys[j];
  if (a == b) return 32 + __clz((uint32_t)(i ^ j));
  return __clz(a ^ b);
}

// Karras 2012: internal node i covers a key range; children are internal
// nodes (>= 0) or leaves (~index in sorted order).
__global__ void k_karras(const uint32_t* __restrict__ keys, int n, int32_t* __restrict__ left,
                         int32_t* __restrict__ right, int32_t* __restrict__ parent_int,
                         int32_t* __restrict__ parent_leaf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int d = (lbvh_delta(keys, n, i, i + 1) - lbvh_delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
  int dmin = lbvh_delta(keys, n, i, i - d);
  int lmax = 2;
  while (lbvh_delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int l = 0;
  for (int t = lmax >> 1; t >= 1; t >>= 1)
    if (lbvh_delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
  int j = i + l * d;
  int dnode = lbvh_delta(keys, n, i, j);
  int s = 0;
  for (int t = (l + 1) >> 1;; t = (t + 1) >> 1) {
    if (lbvh_delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    if (t == 1) break;
  }
  int gamma = i + s * d + (d < 0 ? -1 : 0);
  int lo = min(i, j), hi = max(i, j);
  int L = (lo == gamma) ? ~gamma : gamma;
  int R = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
  left[i] = L;
  right[i] = R;
  if (L >= 0) parent_int[L] = i; else parent_leaf[~L] = i;
  if (R >= 0) parent_int[R] = i; else parent_leaf[~R] = i;
}

// Bottom-up refit: the second thread to reach a node writes both child boxes.
__global__ void k_refit(int n, const int32_t* __restrict__ sorted_ids,
                        const double* __restrict__ leafbox, const int32_t* __restrict__ left,
                        const int32_t* __restrict__ right, const int32_t* __restrict__ parent_int,
                        const int32_t* __restrict__ parent_leaf, int32_t* __restrict__ arrive,
                        double* __restrict__ ibox, Node* __restrict__ nodes) {
  int li = blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= n) return;
  int node = parent_leaf[li];
  while (node >= 0) {
    __threadfence();
    if (atomicAdd(&arrive[node], 1) == 0) return;  // first arrival: sibling not ready
    __threadfence();
    Node nd;
    double u[5] = {INFINITY, -INFINITY, INFINITY, -INFINITY, -INFINITY};
    for (int c = 0; c < 2; ++c) {
      int ch = c == 0 ? left[node] : right[node];
      const double* b;
      if (ch < 0) {
        b = leafbox + 5 * sorted_ids[~ch];
        nd.child[c] = ~sorted_ids[~ch];  // leaf: ~patch id
      } else {
        b = ibox + 5 * ch;
        nd.child[c] = ch;
      }
      double b0 = __ldcg(b), b1 = __ldcg(b + 1), b2 = __ldcg(b + 2), b3 = __ldcg(b + 3),
             b4 = __ldcg(b + 4);
      nd.alo[c] = b0; nd.ahi[c] = b1; nd.blo[c] = b2; nd.bhi[c] = b3; nd.cmax[c] = b4;
      u[0] = fmin(u[0], b0); u[1] = fmax(u[1], b1); u[2] = fmin(u[2], b2);
      u[3] = fmax(u[3], b3); u[4] = fmax(u[4], b4);
    }
    nodes[node] = nd;
    for (int k = 0; k < 5; ++k) __stcg(ibox + 5 * node + k, u[k]);
    node = parent_int[node];
  }
}

// ---- uniform grid over the leaf boxes ------------------------------------

__global__ void k_leaf_extent_sum(const double* __restrict__ leafbox, int64_t n,
                                  double* __restrict__ acc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double w = 0.0, h = 0.0;
  if (i < n) {
    w = leafbox[5 * i + 1] - leafbox[5 * i];
    h = leafbox[5 * i + 3] - leafbox[5 * i + 2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w += __shfl_down_sync(0xffffffffu, w, o);
    h += __shfl_down_sync(0xffffffffu, h, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, w);
    atomicAdd(acc + 1, h);
  }
}

__device__ __forceinline__ void leaf_cells(const double* b, double gx0, double gy0, double gia,
                                           double gib, int ga, int gb, int& i0, int& i1, int& j0,
                                           int& j1) {
  i0 = max(0, min(ga - 1, (int)floor((b[0] - gx0) * gia)));
  i1 = max(0, min(ga - 1, (int)floor((b[1] - gx0) * gia)));
  j0 = max(0, min(gb - 1, (int)floor((b[2] - gy0) * gib)));
  j1 = max(0, min(gb - 1, (int)floor((b[3] - gy0) * gib)));
}

template <bool kFill>
__global__ void k_grid_bin(const double* __restrict__ leafbox, int64_t n, double gx0, double gy0,
                           double gia, double gib, int ga, int gb, int32_t* __restrict__ cnt,
                           const int32_t* __restrict__ offs, CellEnt* __restrict__ cells) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* b = leafbox + 5 * i;
  int i0, i1, j0, j1;
  leaf_cells(b, gx0, gy0, gia, gib, ga, gb, i0, i1, j0, j1);
  CellEnt ent;
  if (kFill) {  // rounded outward: the float test is a superset of the double one
    ent.alo = __double2float_rd(b[0]);
    ent.ahi = __double2float_ru(b[1]);
    ent.blo = __double2float_rd(b[2]);
    ent.bhi = __double2float_ru(b[3]);
    ent.cmax = __double2float_ru(b[4]);
    ent.leaf = (int32_t)i;
  }
  for (int j = j0; j <= j1; ++j)
    for (int ii = i0; ii <= i1; ++ii) {
      const int c = j * ga + ii;
      const int k = atomicAdd(&cnt[c], 1);
      if (kFill) cells[offs[c] + k] = ent;
    }
}

// Build the grid if it stays compact: cell ~ half the mean leaf box extent.
static cudaError_t build_grid(Round& rd, double amin, double amax, double bmin, double bmax,
                              cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  const int64_t n = rd.n_leaves;
  double* acc = nullptr;
  int32_t* cnt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  double h[2] = {0, 0};
  const char* mode = getenv("GWN_CULL");
  if (mode && !strcmp(mode, "bvh")) return cudaSuccess;
#define GC(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)
  GC(cudaMalloc(&acc, 2 * sizeof(double)));
  GC(cudaMemsetAsync(acc, 0, 2 * sizeof(double), st));
  k_leaf_extent_sum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rd.leafbox, n, acc);
  GC(cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, st));
  GC(cudaStreamSynchronize(st));
  {
    // wider than any leaf-box expansion (<= 1e-12 (1 + mag) + 3e-9 patch extent)
    const double margin = 1e-8 * (1.0 + fabs(amin) + fabs(amax) + fabs(bmin) + fabs(bmax));
    const double x0 = amin - margin, x1 = amax + margin, y0 = bmin - margin, y1 = bmax + margin;
    // cell = kf x the mean leaf-box extent (measured best at config 2)
    constexpr double kf = 0.5;
    const double cw = fmax(kf * h[0] / (double)n, (x1 - x0) / 4096.0);
    const double ch = fmax(kf * h[1] / (double)n, (y1 - y0) / 4096.0);
    const int ga = (int)fmin(4096.0, fmax(1.0, ceil((x1 - x0) / cw)));
    const int gb = (int)fmin(4096.0, fmax(1.0, ceil((y1 - y0) / ch)));
    const int64_t ncell = (int64_t)ga * gb;
    if (ncell > (1ll << 24)) goto out;
    rd.ga = ga;
    rd.gb = gb;
    rd.gx0 = x0;
    rd.gy0 = y0;
    rd.gia = ga / (x1 - x0);
    rd.gib = gb / (y1 - y0);
    GC(cudaMalloc(&cnt, sizeof(int32_t) * (ncell + 1)));
    GC(cudaMalloc(&rd.cell_offs, sizeof(int32_t) * (ncell + 1)));
    GC(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ncell + 1), st));
    k_grid_bin<false><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        rd.leafbox, n, rd.gx0, rd.gy0, rd.gia, rd.gib, ga, gb, cnt, nullptr, nullptr);
    GC(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, rd.cell_offs, (int)(ncell + 1), st));
    GC(cudaMalloc(&tmp, tb));
    GC(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, rd.cell_offs, (int)(ncell + 1), st));
    int32_t total = 0;
    GC(cudaMemcpyAsync(&total, rd.cell_offs + ncell, sizeof total, cudaMemcpyDeviceToHost, st));
    GC(cudaStreamSynchronize(st));
    // compact enough?  (else keep the LBVH)
    if (total > 64 * n + 4096 && !(mode && !strcmp(mode, "grid"))) {
      cudaFree(rd.cell_offs);
      rd.cell_offs = nullptr;
      goto out;
    }
    rd.grid_entries = total;
    GC(cudaMalloc(&rd.cell_ent, sizeof(CellEnt) * ((size_t)total + 1)));
    GC(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ncell + 1), st));
    k_grid_bin<true><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        rd.leafbox, n, rd.gx0, rd.gy0, rd.gia, rd.gib, ga, gb, cnt, rd.cell_offs, rd.cell_ent);
    GC(cudaGetLastError());
    GC(cudaStreamSynchronize(st));
    rd.use_grid = true;
    if (getenv("GWN_TRACE"))
      fprintf(stderr, "[gwn] round grid %d x %d, %d entries for %lld leaves (%.2f per cell)\n",
              ga, gb, total, (long long)n, (double)total / ((double)ga * gb));
  }
out:
#undef GC
  if (acc) cudaFree(acc);
  if (cnt) cudaFree(cnt);
  if (tmp) cudaFree(tmp);
  return e;
}

// Grandchild lists of the fold trees: for an internal node t with children
// c0 = t+1 and c1 = t+1+skip[t+1], each child contributes itself if it is a
// leaf, else its two children -- the fallback walks every other level only
// (half the dependent memory round trips) and never skips a leaf.
__global__ void k_foldtree_gc(int64_t total, const int32_t* __restrict__ skip,
                              int4* __restrict__ gc) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  int4 g = make_int4(-1, -1, -1, -1);
  if (skip[t] > 1) {
    const int64_t c[2] = {t + 1, t + 1 + skip[t + 1]};
    int out[4] = {-1, -1, -1, -1};
    int n = 0;
    for (int k = 0; k < 2; ++k) {
      if (skip[c[k]] == 1) {
        out[n++] = (int)(c[k] - t);
      } else {
        out[n++] = (int)(c[k] + 1 - t);
        out[n++] = (int)(c[k] + 1 + skip[c[k] + 1] - t);
      }
    }
    g = make_int4(out[0], out[1], out[2], out[3]);
  }
  gc[t] = g;
}

// Fold trees of the round's uncertified leaves (k_foldtree): the deepest
// sub_level <= kSubLevelMax whose node count stays within the budget
static cudaError_t build_subleaves(Round& rd, cudaStream_t st) {
  int level = kSubLevelMax;
  if (level > kLeafLevelCap) level = kLeafLevelCap;  // (kLeafLevelCap bounds the stacks)
  const int64_t n = rd.n_leaves;
  if (level <= leaf_max_level() || n <= 0) return cudaSuccess;
  const int64_t budget = std::max<int64_t>(4 * n, 1ll << 20);  // node budget
  const int level0 = level;
  double tree_r = kTreeR;  // certified-leaf tree threshold
  cudaError_t e = cudaSuccess;
  int64_t *cnt = nullptr, *offs = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int64_t total = 0;
  const unsigned g = (unsigned)((n + 127) / 128);
#define SC(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)
  SC(cudaMalloc(&cnt, sizeof(int64_t) * (n + 1)));
  SC(cudaMalloc(&offs, sizeof(int64_t) * (n + 1)));
  SC(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs, (int)(n + 1), st));
  SC(cudaMalloc(&tmp, tb));
  {
    // ascending search: the deepest level (and, first, with the wide
    // certified-node splitting) whose node count fits the budget; each
    // deeper count costs ~4x the previous, so the search costs ~1.3 counts
    auto count = [&](int lv, double tr, int64_t& tot) -> cudaError_t {
      cudaError_t ce = cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), st);
      if (ce != cudaSuccess) return ce;
      k_foldtree<false><<<g, 128, 0, st>>>(n, rd.leaves, rd.proj, lv, tr, nullptr, cnt, nullptr,
                                           nullptr, nullptr);
      if ((ce = cudaGetLastError()) != cudaSuccess) return ce;
      if ((ce = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, offs, (int)(n + 1), st)) != cudaSuccess)
        return ce;
      if ((ce = cudaMemcpyAsync(&tot, offs + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st)) !=
          cudaSuccess)
        return ce;
      return cudaStreamSynchronize(st);
    };
    int best = -1;
    bool last_is_best = false;
    const double trs[2] = {tree_r, INFINITY};
    for (int pass = 0; pass < 2 && best < 0; ++pass) {
      if (pass == 1 && !(trs[0] < 1.0)) break;
      int64_t t2 = 0, t1 = 0;  // the two previous counts (growth estimate)
      for (int lv = leaf_max_level() + 2; lv <= level0; lv += 2) {
        // skip a count whose geometric estimate is far over the budget
        if (t2 > 0 && t1 > 0 && (double)t1 * ((double)t1 / (double)t2) > 1.5 * (double)budget)
          break;
        int64_t tot = 0;
        SC(count(lv, trs[pass], tot));
        last_is_best = tot <= budget;
        if (!last_is_best) break;
        best = lv;
        tree_r = trs[pass];
        total = tot;
        t2 = t1;
        t1 = tot;
      }
    }
    if (best < 0) goto out;  // nothing fits: keep the plain fallback
    level = best;
    if (!last_is_best) SC(count(level, tree_r, total));
  }
  if (total > 0) {
    SC(cudaMalloc(&rd.sub, sizeof(LeafRec) * total));
    SC(cudaMalloc(&rd.subbox, sizeof(double) * 5 * total));
    SC(cudaMalloc(&rd.subskip, sizeof(int32_t) * (total + 1)));  // +1: read-ahead pad
    SC(cudaMemsetAsync(rd.subskip + total, 0, sizeof(int32_t), st));
    k_foldtree<true><<<g, 128, 0, st>>>(n, rd.leaves, rd.proj, level, tree_r, offs, nullptr,
                                        rd.sub, rd.subbox, rd.subskip);
    SC(cudaGetLastError());
    SC(cudaMalloc(&rd.subgc, sizeof(int4) * total));
    k_foldtree_gc<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(total, rd.subskip, rd.subgc);
    SC(cudaGetLastError());
    rd.sub_offs = offs;
    offs = nullptr;
    rd.n_sub = total;
    rd.sub_level = level;
    SC(cudaStreamSynchronize(st));
  }
  if (getenv("GWN_TRACE"))
    fprintf(stderr, "[gwn] fold trees: %lld nodes to level %d (certified-leaf trees R >= %g)\n",
            (long long)total, level, tree_r);
out:
#undef SC
  if (cnt) cudaFree(cnt);
  if (offs) cudaFree(offs);
  if (tmp) cudaFree(tmp);
  return e;
}

void free_round(Round& rd) {
  if (rd.sub) cudaFree(rd.sub);
  if (rd.subbox) cudaFree(rd.subbox);
  if (rd.subskip) cudaFree(rd.subskip);
  if (rd.subgc) cudaFree(rd.subgc);
  if (rd.sub_offs) cudaFree(rd.sub_offs);
  if (rd.proj) cudaFree(rd.proj);
  if (rd.powc) cudaFree(rd.powc);
  if (rd.nodes) cudaFree(rd.nodes);
  if (rd.leafbox) cudaFree(rd.leafbox);
  if (rd.leaves) cudaFree(rd.leaves);
  if (rd.vproj) cudaFree(rd.vproj);
  if (rd.ffg) cudaFree(rd.ffg);
  if (rd.ffa) cudaFree(rd.ffa);
  if (rd.ffw) cudaFree(rd.ffw);
  if (rd.ffwg) cudaFree(rd.ffwg);
  if (rd.cell_offs) cudaFree(rd.cell_offs);
  if (rd.cell_ent) cudaFree(rd.cell_ent);
  free_fmm_round(rd);
  rd = Round();
}

// Build the per-direction structures (projection, leaves, cull grid/LBVH,
// boundary vertices in the ray frame) for unit direction d.
cudaError_t build_round_dir(gwn_scene* sc, const double d[3], Round& rd, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  make_frame(d, &rd.f);
  {
    const int64_t P = sc->P;
    if (P > 0) {
      // projected scene bounds from the 8 corners of the scene box
      double amin = INFINITY, amax = -INFINITY, bmin = INFINITY, bmax = -INFINITY;
      for (int c = 0; c < 8; ++c) {
        double x = (c & 1) ? sc->bbox_max[0] : sc->bbox_min[0];
        double y = (c & 2) ? sc->bbox_max[1] : sc->bbox_min[1];
        double z = (c & 4) ? sc->bbox_max[2] : sc->bbox_min[2];
        double A = x * rd.f.e1[0] + y * rd.f.e1[1] + z * rd.f.e1[2];
        double B = x * rd.f.e2[0] + y * rd.f.e2[1] + z * rd.f.e2[2];
        amin = fmin(amin, A); amax = fmax(amax, A);
        bmin = fmin(bmin, B); bmax = fmax(bmax, B);
      }
      double ainv = amax > amin ? 1.0 / (amax - amin) : 0.0;
      double binv = bmax > bmin ? 1.0 / (bmax - bmin) : 0.0;
      rd.amin = amin;
      rd.ainv = ainv;
      rd.bmin = bmin;
      rd.binv = binv;
      uint32_t *keys = nullptr, *keys2 = nullptr;
      int32_t *ids = nullptr, *ids2 = nullptr, *tmp = nullptr;
      int64_t *lcount = nullptr, *loffs = nullptr;
      double* ibox = nullptr;
      void* cub_tmp = nullptr;
      size_t cub_bytes = 0;
      int64_t nl = 0;
      int n = 0;
      unsigned lb = 0;
      const unsigned pb = (unsigned)((P + 127) / 128);
#define RC(x)                     \
  do {                            \
    e = (x);                      \
    if (e != cudaSuccess) goto out; \
  } while (0)
      RC(cudaMalloc(&rd.proj, sizeof(double) * 48 * P));
      RC(cudaMalloc(&rd.powc, sizeof(double) * 48 * P));
      k_project<<<pb, 128, 0, st>>>(sc->ctrl, P, rd.f, rd.proj, rd.powc);
      RC(cudaGetLastError());
      // leaves: count, scan, fill
      RC(cudaMalloc(&lcount, sizeof(int64_t) * (P + 1)));
      RC(cudaMalloc(&loffs, sizeof(int64_t) * (P + 1)));
      RC(cudaMemsetAsync(lcount + P, 0, sizeof(int64_t), st));
      k_leaves<false><<<(unsigned)((P + 63) / 64), 64, 0, st>>>(
          P, rd.proj, nullptr, lcount, nullptr, nullptr, nullptr, nullptr, amin, ainv, bmin, binv, leaf_max_level());
      RC(cudaGetLastError());
      RC(cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, lcount, loffs, (int)P + 1, st));
      RC(cudaMalloc(&cub_tmp, cub_bytes));
      RC(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, lcount, loffs, (int)P + 1, st));
      RC(cudaMemcpyAsync(&nl, loffs + P, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      RC(cudaStreamSynchronize(st));
      cudaFree(cub_tmp);
      cub_tmp = nullptr;
      cub_bytes = 0;
      if (nl <= 0 || nl > (1ll << 30)) {
        e = cudaErrorInvalidValue;
        goto out;
      }
      rd.n_leaves = nl;
      n = (int)nl;
      lb = (unsigned)((nl + 127) / 128);
      RC(cudaMalloc(&rd.leaves, sizeof(LeafRec) * nl));
      RC(cudaMalloc(&rd.leafbox, sizeof(double) * 5 * nl));
      RC(cudaMalloc(&keys, sizeof(uint32_t) * nl));
      RC(cudaMalloc(&keys2, sizeof(uint32_t) * nl));
      RC(cudaMalloc(&ids, sizeof(int32_t) * nl));
      RC(cudaMalloc(&ids2, sizeof(int32_t) * nl));
      k_leaves<true><<<(unsigned)((P + 63) / 64), 64, 0, st>>>(
          P, rd.proj, loffs, nullptr, rd.leaves, rd.leafbox, keys, ids, amin, ainv, bmin, binv, leaf_max_level());
      RC(cudaGetLastError());
      if (nl > 1) {
        RC(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, keys, keys2, ids, ids2, n, 0, 30,
                                           st));
        RC(cudaMalloc(&cub_tmp, cub_bytes));
        RC(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, keys2, ids, ids2, n, 0, 30,
                                           st));
        RC(cudaMalloc(&rd.nodes, sizeof(Node) * (nl - 1)));
        RC(cudaMalloc(&tmp, sizeof(int32_t) * (5 * nl)));
        RC(cudaMalloc(&ibox, sizeof(double) * 5 * (nl - 1)));
        {
          int32_t* left = tmp;
          int32_t* right = tmp + nl;
          int32_t* parent_int = tmp + 2 * nl;
          int32_t* parent_leaf = tmp + 3 * nl;
          int32_t* arrive = tmp + 4 * nl;
          RC(cudaMemsetAsync(arrive, 0, sizeof(int32_t) * nl, st));
          RC(cudaMemsetAsync(parent_int, 0xff, sizeof(int32_t) * nl, st));  // root parent = -1
          k_karras<<<lb, 128, 0, st>>>(keys2, n, left, right, parent_int, parent_leaf);
          RC(cudaGetLastError());
          k_refit<<<lb, 128, 0, st>>>(n, ids2, rd.leafbox, left, right, parent_int, parent_leaf,
                                      arrive, ibox, rd.nodes);
          RC(cudaGetLastError());
        }
      }
      RC(cudaStreamSynchronize(st));
      RC(build_grid(rd, amin, amax, bmin, bmax, st));
      // First guess of the candidates per query from the grid's fill (config 5:
      // 14.9 entries per cell, 7.9 candidates per query).  With the default of
      // 4 the first eval of a dense scene overflowed its candidate buffer:
      // round 0 ran twice and the 30 GB K3 scratch was re-allocated, 0.75 s of
      // a 1.5 s first eval.  A wrong guess still only costs that, or memory.
      if (rd.use_grid && sc->pairs_per_query == 4.0 && !getenv("GWN_PAIRS_INIT"))
        sc->pairs_per_query =
            fmax(4.0, 0.55 * (double)rd.grid_entries / ((double)rd.ga * (double)rd.gb));
      RC(build_subleaves(rd, st));
    out:
      if (keys) cudaFree(keys);
      if (keys2) cudaFree(keys2);
      if (ids) cudaFree(ids);
      if (ids2) cudaFree(ids2);
      if (tmp) cudaFree(tmp);
      if (ibox) cudaFree(ibox);
      if (cub_tmp) cudaFree(cub_tmp);
      if (lcount) cudaFree(lcount);
      if (loffs) cudaFree(loffs);
#undef RC
      if (e != cudaSuccess) {
        free_round(rd);
        return e;
      }
    }
    if ((e = launch_vproj(sc, rd, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess) {
      free_round(rd);
      return e;
    }
  }
  return e;
}

// Caller holds sc->mu.  Builds rounds[0..r] that are missing.
cudaError_t build_round(gwn_scene* sc, int r, cudaStream_t st) {
  while ((int)sc->rounds.size() <= r) {
    double d[3];
    gwn_direction(sc->prm.dir_seed, (int32_t)sc->rounds.size(), d);
    Round rd;
    cudaError_t e = build_round_dir(sc, d, rd, st);
    if (e != cudaSuccess) return e;
    sc->rounds.push_back(rd);
  }
  return cudaSuccess;
}

}  // namespace gwn
