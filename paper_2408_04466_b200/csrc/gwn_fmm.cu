// gwn_fmm.cu -- local expansions of the boundary term's far field (K4).
//
// The per-pair far field (gwn_boundary.cu, k_ff_fill) evaluates, for every
// query, the multipole expansion of every far closed cycle: ~840 expansions
// of ~73 terms per query at config 5, 71% of the step.  Here the cycles'
// multipoles are translated once per direction round into local expansions
// on an octree over the scene cube, so a query evaluates ONE order-kFmmP local
// expansion (its leaf's) plus the few cycles its leaf could not take.
//
// Math (solid harmonics R, I and moments D as in gwn_farfield.cuh; checked in
// tools/farfield/fmm_proto.py):
//   M2L  I_n^m(b + x) = sum_{j,k} (-1)^j conj(R_j^k(x)) I_{n+j}^{m+k}(b), |x| < |b|, so
//        Omega(z + x) = sum_{j,k} conj(R_j^k(x)) L_j^k with
//        L_j^k = -(-1)^j sum_{n=1..K} sum_{m=-n..n} D_n^m I_{n+j}^{m+k}(z - g);
//   L2L  R_n^m(x + y) = sum_{a,b} R_a^b(x) R_{n-a}^{m-b}(y) gives the child's
//        L'_a^b = sum_{j>=a} sum_k conj(R_{j-a}^{k-b}(y)) L_j^k, exact (a degree-P
//        polynomial re-centred);
//   L2P  fmm_l2p (gwn_farfield.cuh).
// Negative orders by X_n^{-m} = (-1)^m conj(X_n^m) for X = R, I, D, L.
//
// Error budget of a translated (box, cycle) pair, each half tau / 2 (tau:
// the scene's per-entry share, gwn_farfield.cu):
//   (1) the cycle's multipole truncated at K = kFmmK (the orders M2L
//       translates) at the box's nearest point, D - r_B:
//       ff_bound(A_abs, rho, K, D - r_B);
//   (2) the order-P local truncation: Omega_K is harmonic in the ball B(z, R0)
//       for R0 < D - rho; with M = max |Omega_K| there, the degree-j part obeys
//       |u_j(x)| <= (2j+1) M (|x|/R0)^j (Poisson kernel, |P_j| <= 1), so the tail
//       past P is <= M (2P+3) t^(P+1) / (1-t)^2 with t = r_B / R0, and
//       M <= A_abs / (D - R0 - rho)^2 + ff_bound(A_abs, rho, K, D - R0).
// Both decrease in the box-centre distance D, so fmm_setup_scene tabulates per
// (cycle, level) the smallest D meeting both (bisection, best of several R0):
// the per-pair guarantee equals the per-pair path's (tau).  The line test
// of the per-pair path (the line through the query misses the cycle's sphere)
// holds for every query of a box when the line through its centre passes the
// sphere by more than the box's circumradius.
//
// Slivers (edges closed by their chord) keep their exact chord term per query
// and exact-only entries have no expansion: both stay on every leaf's
// leftover list, as does every cycle no ancestor box took.
#include <cub/cub.cuh>
#include <math.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "gwn_farfield.cuh"

namespace gwn {

#ifndef GWN_FMM_MAXL
#define GWN_FMM_MAXL 6
#endif
#ifndef GWN_FMM_LEAF
#define GWN_FMM_LEAF 0.6
#endif
constexpr int kFmmMaxL = GWN_FMM_MAXL;  // 8^6 = 262,144 leaves, ~1.4 GB of coefficients
constexpr int kFmmMinCycles = 32;  // fewer closed cycles: the per-pair path alone

// ---------------------------------------------------------------------------
// scene level: the cube, the leaf level and the acceptance distances
// ---------------------------------------------------------------------------

static double fmm_tail_bound(double aabs, double rho, double rB, double D) {
  double best = INFINITY;
  for (int i = 1; i <= 9; ++i) {  // R0 between r_B and D - rho
    const double R0 = rB + (D - rho - rB) * (0.1 * i);
    if (!(R0 > rB) || !(D - R0 - rho > 0.0)) continue;
    const double M = aabs / ((D - R0 - rho) * (D - R0 - rho)) + ff_bound(aabs, rho, kFmmK, D - R0);
    const double t = rB / R0;
    const double tail = M * (2.0 * kFmmP + 3.0) * pow(t, kFmmP + 1.0) / ((1.0 - t) * (1.0 - t));
    best = fmin(best, tail);
  }
  return best;
}

static bool fmm_ok(double aabs, double rho, double rB, double D, double half_tau) {
  if (!(D - rB > rho)) return false;
  return ff_bound(aabs, rho, kFmmK, D - rB) <= half_tau &&
         fmm_tail_bound(aabs, rho, rB, D) <= half_tau;
}

static double fmm_box_radius(const gwn_scene* sc, int l) {
  const double h = sc->fmm_side / (double)(1 << l);
  // circumradius, widened for the rounding of a query's leaf index
  return 0.8660254037844387 * h * (1.0 + 1e-9) + 1e-12 * sc->fmm_side;
}

cudaError_t fmm_setup_scene(gwn_scene* sc, const std::vector<double>& rho,
                            const std::vector<double>& aabs, const std::vector<char>& closed) {
  sc->fmm_L = 0;
  const int nk = sc->ff_n;
  std::vector<double> rc;
  for (int c = 0; c < nk; ++c)
    if (closed[c]) rc.push_back(rho[c]);
  if ((int)rc.size() < kFmmMinCycles) return cudaSuccess;
  std::nth_element(rc.begin(), rc.begin() + rc.size() / 2, rc.end());
  const double med = rc[rc.size() / 2];
  double ext = 0.0;
  for (int k = 0; k < 3; ++k) ext = fmax(ext, sc->bbox_max[k] - sc->bbox_min[k]);
  sc->fmm_side = ext * (1.0 + 1e-7) + 1e-12;
  for (int k = 0; k < 3; ++k)
    sc->fmm_x0[k] = 0.5 * (sc->bbox_min[k] + sc->bbox_max[k]) - 0.5 * sc->fmm_side;
  // leaf side ~0.6 of the median cycle radius (measured best trade between
  // translations and leftover pairs at config 5)
  const int L = (int)ceil(log2(sc->fmm_side / (GWN_FMM_LEAF * med)));
  sc->fmm_L = std::max(2, std::min(kFmmMaxL, L));
  const int nl = sc->fmm_L + 1;
  std::vector<double> dmin((size_t)nk * nl, INFINITY);
  for (int c = 0; c < nk; ++c) {
    if (!closed[c]) continue;
    for (int l = 0; l < nl; ++l) {
      const double rB = fmm_box_radius(sc, l);
      double lo = rB + rho[c], hi = 2.0 * lo + 1.0;
      int guard = 0;
      while (!fmm_ok(aabs[c], rho[c], rB, hi, 0.5 * sc->ff_tau) && guard++ < 200) hi *= 2.0;
      if (guard >= 200) continue;
      for (int it = 0; it < 80; ++it) {
        const double mid = 0.5 * (lo + hi);
        (fmm_ok(aabs[c], rho[c], rB, mid, 0.5 * sc->ff_tau) ? hi : lo) = mid;
      }
      dmin[(size_t)c * nl + l] = hi;
    }
  }
  cudaError_t e = cudaMalloc(&sc->fmm_dmin, sizeof(double) * dmin.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->fmm_dmin, dmin.data(), sizeof(double) * dmin.size(),
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (sc->fmm_dmin) cudaFree(sc->fmm_dmin);
    sc->fmm_dmin = nullptr;
    sc->fmm_L = 0;
  }
  return e;
}

// ---------------------------------------------------------------------------
// round level: acceptance masks, interaction lists, M2L + L2L, leftover lists
// ---------------------------------------------------------------------------

struct FmmGeo {
  int l, n;          // level, boxes per axis
  double x0, y0, z0, h;
  double rB;
  int32_t C, W;      // entries, mask words
  int nl;            // levels in the dmin table
  double dx, dy, dz; // round direction (world)
};

__device__ __forceinline__ void fmm_centre(const FmmGeo& G, int64_t b, double& zx, double& zy,
                                           double& zz) {
  const int64_t n = G.n;
  const int64_t ix = b / (n * n), iy = (b / n) % n, iz = b % n;
  zx = G.x0 + ((double)ix + 0.5) * G.h;
  zy = G.y0 + ((double)iy + 0.5) * G.h;
  zz = G.z0 + ((double)iz + 0.5) * G.h;
}

__device__ __forceinline__ int64_t fmm_parent(const FmmGeo& G, int64_t b) {
  const int64_t n = G.n, np = n >> 1;
  const int64_t ix = b / (n * n), iy = (b / n) % n, iz = b % n;
  return ((ix >> 1) * np + (iy >> 1)) * np + (iz >> 1);
}

// One thread per box: acceptance bits of the level (acc), bits its ancestors
// already took (cons), and the counts of new translations / leftover entries.
__global__ void k_fmm_accept(FmmGeo G, const double* __restrict__ g, const double* __restrict__ r2,
                             const double* __restrict__ dmin, const uint32_t* __restrict__ acc_up,
                             const uint32_t* __restrict__ cons_up, uint32_t* __restrict__ acc,
                             uint32_t* __restrict__ cons, int32_t* __restrict__ n_new,
                             int32_t* __restrict__ n_left) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nb = (int64_t)G.n * G.n * G.n;
  if (b >= nb) return;
  double zx, zy, zz;
  fmm_centre(G, b, zx, zy, zz);
  const int64_t p = G.l > 0 ? fmm_parent(G, b) : 0;
  int32_t cnt_new = 0, cnt_left = 0;
  for (int w = 0; w < G.W; ++w) {
    uint32_t a = 0;
    for (int i = 0; i < 32; ++i) {
      const int c = w * 32 + i;
      if (c >= G.C) break;
      const double dm = __ldg(dmin + (int64_t)c * G.nl + G.l);
      if (!(dm < INFINITY)) continue;
      const double vx = zx - __ldg(g + 3 * c), vy = zy - __ldg(g + 3 * c + 1),
                   vz = zz - __ldg(g + 3 * c + 2);
      const double D2 = vx * vx + vy * vy + vz * vz;
      if (D2 < dm * dm) continue;
      // the forward half-lines p + t d of the box's points miss the sphere
      // (ff_far2's line test for every p in the box): the line through the
      // centre passes it by more than r_B, or the sphere lies wholly behind
      // the box along d
      const double t = vx * G.dx + vy * G.dy + vz * G.dz;  // (z - g) . d
      const double lr = sqrt(__ldg(r2 + 2 * c + 1)) + G.rB;
      if (D2 - t * t <= lr * lr && !(t > lr)) continue;
      a |= 1u << i;
    }
    const uint32_t cu = G.l > 0 ? (cons_up[p * G.W + w] | acc_up[p * G.W + w]) : 0u;
    acc[b * G.W + w] = a;
    cons[b * G.W + w] = cu;
    cnt_new += __popc(a & ~cu);
    uint32_t valid = G.C - w * 32 >= 32 ? 0xffffffffu : ((1u << (G.C - w * 32)) - 1u);
    cnt_left += __popc(~(a | cu) & valid);
  }
  n_new[b] = cnt_new;
  if (n_left) n_left[b] = cnt_left;
}

// lists in ascending entry order: mode 0 = new translations (acc & ~cons),
// mode 1 = leftover (~(acc | cons))
__global__ void k_fmm_lists(int64_t nb, int32_t C, int32_t W, const uint32_t* __restrict__ acc,
                            const uint32_t* __restrict__ cons, const int32_t* __restrict__ off,
                            int32_t* __restrict__ ent, int mode) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int32_t o = off[b];
  for (int w = 0; w < W; ++w) {
    const uint32_t a = acc[b * W + w], cu = cons[b * W + w];
    const uint32_t valid = C - w * 32 >= 32 ? 0xffffffffu : ((1u << (C - w * 32)) - 1u);
    uint32_t bits = mode == 0 ? (a & ~cu) : (~(a | cu) & valid);
    while (bits) {
      const int i = __ffs(bits) - 1;
      bits &= bits - 1;
      ent[o++] = w * 32 + i;
    }
  }
}

// the outside list (queries beyond the cube): every entry
__global__ void k_fmm_all(int32_t C, int32_t* __restrict__ ent) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) ent[c] = c;
}

constexpr int kM2LThreads = 256;

// conj-and-sign access for a negative order: X_n^{-m} = (-1)^m conj(X_n^m)
__device__ __forceinline__ double2 fmm_get(const double2* __restrict__ T, int n, int m) {
  const int am = m < 0 ? -m : m;
  double2 v = T[ff_term(n, am)];
  if (m < 0) {
    v.y = -v.y;
    if (am & 1) {
      v.x = -v.x;
      v.y = -v.y;
    }
  }
  return v;
}

// Shared tables of the M2L block, every order m in [-n, n] stored (row n at
// n^2, order m at n^2 + n + m) so the inner loop walks both with unit stride
// and no sign logic: I_N^M(b) for N <= kFmmIN and the entry's D_n^m, n <= kFmmK.
constexpr int kFmmIFull = (kFmmIN + 1) * (kFmmIN + 1);
constexpr int kFmmDFull = (kFmmK + 1) * (kFmmK + 1);
constexpr size_t kM2LSmem = sizeof(double2) * (kFmmIFull + kFmmDFull + kFmmLT);

__device__ __forceinline__ double2 fmm_neg(double2 v, int m) {  // X_n^{-m} from X_n^m
  return (m & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
}

// One block per box of level l: the L2L of the parent's expansion (l > 0)
// plus the M2L of every cycle on the box's list; thread t < kFmmLT owns the
// coefficient (j, k) with t = j (j+1)/2 + k.
__global__ void __launch_bounds__(kM2LThreads)
k_fmm_m2l(FmmGeo G, const int32_t* __restrict__ off, const int32_t* __restrict__ ent,
          const double* __restrict__ g, const double2* __restrict__ D,
          const double2* __restrict__ Lup, double2* __restrict__ Lout) {
  extern __shared__ double2 sm[];
  double2* sI = sm;                    // (kFmmIN+1)^2, full orders
  double2* sD = sm + kFmmIFull;        // (kFmmK+1)^2, full orders
  double2* sL = sD + kFmmDFull;        // parent's L_j^k, k >= 0
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  int j = 0;
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  const int k = t - j * (j + 1) / 2;
  const bool own = t < kFmmLT;
  double zx, zy, zz;
  fmm_centre(G, b, zx, zy, zz);
  double aR = 0.0, aI = 0.0;
  if (G.l > 0) {
    // L2L from the parent: y = z - z_parent, its regular harmonics in sI
    // (orders m >= 0 at ff_term(n, m))
    const int64_t p = fmm_parent(G, b);
    FmmGeo Gp = G;
    Gp.n = G.n >> 1;
    Gp.h = 2.0 * G.h;
    double px, py, pz;
    fmm_centre(Gp, p, px, py, pz);
    const double x = zx - px, y = zy - py, z = zz - pz, r2 = x * x + y * y + z * z;
    for (int q = t; q < kFmmLT; q += blockDim.x) sL[q] = Lup[p * kFmmLT + q];
    if (t <= kFmmP) {  // column m = t of R_n^m(y), n <= P
      const int m = t;
      double dR = 1.0, dI = 0.0;
      for (int i = 1; i <= m; ++i) {
        const double c0 = -1.0 / (2.0 * i);
        const double nR = c0 * (x * dR - y * dI), nI = c0 * (x * dI + y * dR);
        dR = nR;
        dI = nI;
      }
      double vR = dR, vI = dI, uR = 0.0, uI = 0.0;
      sI[ff_term(m, m)] = make_double2(vR, vI);
      for (int n = m + 1; n <= kFmmP; ++n) {
        const double inv = 1.0 / ((double)(n + m) * (double)(n - m));
        const double k1 = (2.0 * n - 1.0) * z;
        const double wR = (k1 * vR - r2 * uR) * inv, wI = (k1 * vI - r2 * uI) * inv;
        uR = vR;
        uI = vI;
        vR = wR;
        vI = wI;
        sI[ff_term(n, m)] = make_double2(vR, vI);
      }
    }
    __syncthreads();
    if (own) {
      // L'_j^k = sum_{a >= j} sum_c conj(R_{a-j}^{c-k}(y)) L_a^c
      for (int a = j; a <= kFmmP; ++a) {
        const int na = a - j;
        const int c_lo = max(-a, k - na), c_hi = min(a, k + na);
        for (int c = c_lo; c <= c_hi; ++c) {
          const double2 r = fmm_get(sI, na, c - k);
          const double2 l = fmm_get(sL, a, c);
          // conj(r) * l
          aR = fma(r.x, l.x, fma(r.y, l.y, aR));
          aI = fma(r.x, l.y, fma(-r.y, l.x, aI));
        }
      }
    }
  }
  const int32_t e0 = off[b], e1 = off[b + 1];
  for (int32_t e = e0; e < e1; ++e) {
    const int c = ent[e];
    __syncthreads();  // previous tables consumed
    for (int q = t; q < kFmmKT; q += blockDim.x) {  // D_n^m, both signs of m
      int n = 0;
      while ((n + 1) * (n + 2) / 2 <= q) ++n;
      const int m = q - n * (n + 1) / 2;
      const double2 v = D[(int64_t)c * kFFTerms + q];
      sD[n * n + n + m] = v;
      sD[n * n + n - m] = m ? fmm_neg(v, m) : v;
    }
    const double x = zx - __ldg(g + 3 * c), y = zy - __ldg(g + 3 * c + 1),
                 z = zz - __ldg(g + 3 * c + 2);
    if (t <= kFmmIN) {  // column m = t of I_n^m(b), n <= K + P, and its mirror -m
      const int m = t;
      const double ir2 = 1.0 / (x * x + y * y + z * z);
      double dR = sqrt(ir2), dI = 0.0;
      for (int i = 1; i <= m; ++i) {
        const double c0 = -(2.0 * i - 1.0) * ir2;
        const double nR = c0 * (x * dR - y * dI), nI = c0 * (x * dI + y * dR);
        dR = nR;
        dI = nI;
      }
      double vR = dR, vI = dI, uR = 0.0, uI = 0.0;
      for (int n = m;; ++n) {
        const double2 v = make_double2(vR, vI);
        sI[n * n + n + m] = v;
        sI[n * n + n - m] = m ? fmm_neg(v, m) : v;
        if (n == kFmmIN) break;
        const double kz = (2.0 * n + 1.0) * z;
        const double k2 = (double)(n * n - m * m);
        const double wR = (kz * vR - k2 * uR) * ir2, wI = (kz * vI - k2 * uI) * ir2;
        uR = vR;
        uI = vI;
        vR = wR;
        vI = wI;
      }
    }
    __syncthreads();
    if (own) {
      // sum_{n, m} D_n^m I_{n+j}^{m+k}: two accumulator pairs (even / odd m)
      double sR0 = 0.0, sI0 = 0.0, sR1 = 0.0, sI1 = 0.0;
      for (int n = 1; n <= kFmmK; ++n) {
        const double2* Dn = sD + n * n;                       // m = -n at Dn[0]
        const double2* In = sI + (n + j) * (n + j) + j + k;   // I_{n+j}^{m+k}, m = -n at In[0]
        const int len = 2 * n + 1;
        int q = 0;
        for (; q + 1 < len; q += 2) {
          const double2 d0 = Dn[q], i0 = In[q], d1 = Dn[q + 1], i1 = In[q + 1];
          sR0 = fma(d0.x, i0.x, fma(-d0.y, i0.y, sR0));
          sI0 = fma(d0.x, i0.y, fma(d0.y, i0.x, sI0));
          sR1 = fma(d1.x, i1.x, fma(-d1.y, i1.y, sR1));
          sI1 = fma(d1.x, i1.y, fma(d1.y, i1.x, sI1));
        }
        const double2 d0 = Dn[q], i0 = In[q];
        sR0 = fma(d0.x, i0.x, fma(-d0.y, i0.y, sR0));
        sI0 = fma(d0.x, i0.y, fma(d0.y, i0.x, sI0));
      }
      const double sgn = (j & 1) ? 1.0 : -1.0;  // -(-1)^j
      aR = fma(sgn, sR0 + sR1, aR);
      aI = fma(sgn, sI0 + sI1, aI);
    }
  }
  if (own) Lout[b * kFmmLT + t] = make_double2(aR, aI);
}

void free_fmm_round(Round& rd) {
  if (!rd.fmm) return;
  if (rd.fmm->leafL) cudaFree(rd.fmm->leafL);
  if (rd.fmm->loff) cudaFree(rd.fmm->loff);
  if (rd.fmm->lent) cudaFree(rd.fmm->lent);
  delete rd.fmm;
  rd.fmm = nullptr;
}

cudaError_t build_fmm_round(const gwn_scene* sc, Round& rd, cudaStream_t st) {
  if (rd.fmm || sc->fmm_L <= 0 || sc->ff_n <= 0) return cudaSuccess;
  const auto t0 = std::chrono::steady_clock::now();
  const int L = sc->fmm_L;
  const int32_t C = sc->ff_n, W = (C + 31) / 32;
  const int64_t nleaf = (int64_t)1 << (3 * L);
  FmmRound* F = new FmmRound();
  F->L = L;
  F->n_leaf = nleaf;
  uint32_t *acc[2] = {nullptr, nullptr}, *cons[2] = {nullptr, nullptr};
  int32_t *cnt = nullptr, *off = nullptr, *ent = nullptr, *lcnt = nullptr;
  double2* Lb[2] = {nullptr, nullptr};
  void* tmp = nullptr;
  size_t tmp_bytes = 0, ent_cap = 0;
  int32_t* h = nullptr;
  cudaError_t e = cudaSuccess;
#define FM(x)                        \
  do {                               \
    if ((e = (x)) != cudaSuccess) goto out; \
  } while (0)
  FM(cudaFuncSetAttribute(k_fmm_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)kM2LSmem));
  FM(cudaMallocHost(&h, 2 * sizeof(int32_t)));
  for (int i = 0; i < 2; ++i) {
    FM(cudaMalloc(&acc[i], sizeof(uint32_t) * nleaf * W));
    FM(cudaMalloc(&cons[i], sizeof(uint32_t) * nleaf * W));
    FM(cudaMalloc(&Lb[i], sizeof(double2) * nleaf * kFmmLT));
  }
  FM(cudaMalloc(&cnt, sizeof(int32_t) * (nleaf + 1)));
  FM(cudaMalloc(&lcnt, sizeof(int32_t) * (nleaf + 2)));
  FM(cudaMalloc(&off, sizeof(int32_t) * (nleaf + 1)));
  FM(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, (int)nleaf + 2, st));
  FM(cudaMalloc(&tmp, tmp_bytes));
  for (int l = 0; l <= L; ++l) {
    const int cur = l & 1, up = cur ^ 1;
    const int64_t nb = (int64_t)1 << (3 * l);
    FmmGeo G;
    G.l = l;
    G.n = 1 << l;
    G.x0 = sc->fmm_x0[0];
    G.y0 = sc->fmm_x0[1];
    G.z0 = sc->fmm_x0[2];
    G.h = sc->fmm_side / (double)G.n;
    G.rB = fmm_box_radius(sc, l);
    G.C = C;
    G.W = W;
    G.nl = L + 1;
    G.dx = rd.f.d[0];
    G.dy = rd.f.d[1];
    G.dz = rd.f.d[2];
    const unsigned gb = (unsigned)((nb + 127) / 128);
    k_fmm_accept<<<gb, 128, 0, st>>>(G, sc->ff_g, sc->ff_r, sc->fmm_dmin, acc[up], cons[up],
                                     acc[cur], cons[cur], cnt, l == L ? lcnt : nullptr);
    FM(cudaGetLastError());
    FM(cudaMemsetAsync(cnt + nb, 0, sizeof(int32_t), st));
    FM(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, (int)nb + 1, st));
    FM(cudaMemcpyAsync(h, off + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FM(cudaStreamSynchronize(st));
    const size_t npair = (size_t)h[0];
    F->m2l_pairs += (int64_t)npair;
    if (npair + 1 > ent_cap) {
      if (ent) cudaFree(ent);
      ent = nullptr;
      ent_cap = npair + npair / 4 + 1024;
      FM(cudaMalloc(&ent, sizeof(int32_t) * ent_cap));
    }
    k_fmm_lists<<<gb, 128, 0, st>>>(nb, C, W, acc[cur], cons[cur], off, ent, 0);
    FM(cudaGetLastError());
    k_fmm_m2l<<<(unsigned)nb, kM2LThreads, kM2LSmem, st>>>(G, off, ent, sc->ff_g,
                                                     reinterpret_cast<const double2*>(sc->ff_D),
                                                     Lb[up], Lb[cur]);
    FM(cudaGetLastError());
    if (l == L) {
      // leftover lists of the leaves, then the outside list (every entry)
      FM(cudaMemcpyAsync(lcnt + nleaf, &C, sizeof(int32_t), cudaMemcpyHostToDevice, st));
      FM(cudaMalloc(&F->loff, sizeof(int32_t) * (nleaf + 2)));
      FM(cudaMemsetAsync(lcnt + nleaf + 1, 0, sizeof(int32_t), st));
      FM(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, lcnt, F->loff, (int)nleaf + 2, st));
      FM(cudaMemcpyAsync(h + 1, F->loff + nleaf + 1, sizeof(int32_t), cudaMemcpyDeviceToHost,
                         st));
      FM(cudaStreamSynchronize(st));
      F->leftover = (int64_t)h[1] - C;
      FM(cudaMalloc(&F->lent, sizeof(int32_t) * ((size_t)h[1] + 1)));
      k_fmm_lists<<<gb, 128, 0, st>>>(nleaf, C, W, acc[cur], cons[cur], F->loff, F->lent, 1);
      FM(cudaGetLastError());
      // the outside list starts at loff[nleaf]
      {
        int32_t o = 0;
        FM(cudaMemcpyAsync(&o, F->loff + nleaf, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        FM(cudaStreamSynchronize(st));
        k_fmm_all<<<(C + 255) / 256, 256, 0, st>>>(C, F->lent + o);
        FM(cudaGetLastError());
      }
      F->leafL = Lb[cur];
      Lb[cur] = nullptr;
    }
  }
  FM(cudaStreamSynchronize(st));
  F->ms_build =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  rd.fmm = F;
  F = nullptr;
out:
#undef FM
  for (int i = 0; i < 2; ++i) {
    if (acc[i]) cudaFree(acc[i]);
    if (cons[i]) cudaFree(cons[i]);
    if (Lb[i]) cudaFree(Lb[i]);
  }
  if (cnt) cudaFree(cnt);
  if (lcnt) cudaFree(lcnt);
  if (off) cudaFree(off);
  if (ent) cudaFree(ent);
  if (tmp) cudaFree(tmp);
  if (h) cudaFreeHost(h);
  if (F) {
    Round tmpr;
    tmpr.fmm = F;
    free_fmm_round(tmpr);
  }
  return e;
}

}  // namespace gwn
