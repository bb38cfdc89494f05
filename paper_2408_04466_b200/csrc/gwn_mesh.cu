// gwn_mesh.cu -- the rest of the reference's kernel dispatch layer
// (pkg/src/gwn/_kernels.py) on the B200: triangle-mesh solid-angle sums,
// and all-hits ray/mesh intersection.  (Great-circle arc crossings, the
// generic arrangement's primitive, are out of scope: SURVEY.md §2.)
//
// Semantics follow the reference's numpy twins, which are correct; the
// numba kernels share the broken _cross helper (_kernels.py:45).
//   * solid_angle_many / solid_angle_sum (_kernels.py:385-475): per query the
//     van Oosterom-Strackee sum of 2 atan2(num, den) over the triangles,
//     leaving out (and flagging) triangles the query is on (:405-411).
//     B200: query tiles x triangle tiles staged in shared memory, the
//     per-triangle atan2 replaced by the running complex product of
//     gwn_fan.cuh (one atan2 per query), rsqrt by MUFU seed + Halley.
//   * bvh_ray_all_hits (_kernels.py:366-381) on the reference's Bvh arrays
//     (surfaces.py:74-163) for a batch of rays: Moller-Trumbore with the
//     parallel-ray tangent-contact rule of _ray_tris_hits_numpy (:312-363).
//     One thread per ray walks the BVH with a slab test widened by the largest
//     circumradius (never cull a hit or tangent contact the brute-force twin
//     finds -- the reference's own BVH walk can); count pass, scan,
//     fill pass, then one radix sort of (ray, kind, triangle) puts every
//     ray's hits in the numpy twin's order (regular hits by triangle, then
//     parallel contacts by triangle).
#include <cub/cub.cuh>

#include <math.h>
#include <string.h>

#include <vector>

#include "gwn_fan.cuh"

namespace gwn {

// ---------------------------------------------------------------------------
// solid angles
// ---------------------------------------------------------------------------

constexpr int kTileT = 512;     // triangles per shared tile (9 x 512 x 8 B = 36 KB)
constexpr int kSaBlock = 256;   // queries per block (2 per thread)

__global__ void k_tri_gather(const double* __restrict__ V, const int64_t* __restrict__ T,
                             int64_t nT, int64_t nV, double* __restrict__ tri,
                             int* __restrict__ bad) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nT) return;
  for (int c = 0; c < 3; ++c) {
    const int64_t vi = T[3 * f + c];
    if (vi < 0 || vi >= nV) {
      *bad = 1;
      for (int k = 0; k < 3; ++k) tri[(int64_t)(3 * c + k) * nT + f] = 0.0;
      continue;
    }
    for (int k = 0; k < 3; ++k) tri[(int64_t)(3 * c + k) * nT + f] = V[3 * vi + k];
  }
}

struct SaAcc {
  SegState st;
  int n;
  bool on;
};

__device__ __forceinline__ void sa_term(SaAcc& acc, double px, double py, double pz,
                                        const double* t, double guard2, double guard) {
  const double ax = t[0] - px, ay = t[1] - py, az = t[2] - pz;
  const double bx = t[3] - px, by = t[4] - py, bz = t[5] - pz;
  const double cx = t[6] - px, cy = t[7] - py, cz = t[8] - pz;
  const double a2 = ax * ax + ay * ay + az * az;
  const double b2 = bx * bx + by * by + bz * bz;
  const double c2 = cx * cx + cy * cy + cz * cz;
  if (a2 < guard2 || b2 < guard2 || c2 < guard2) {  // |a| < guard (:399)
    acc.on = true;
    return;
  }
  const double la = a2 * rsqrt_nr(a2), lb = b2 * rsqrt_nr(b2), lc = c2 * rsqrt_nr(c2);
  const double crx = by * cz - bz * cy, cry = bz * cx - bx * cz, crz = bx * cy - by * cx;
  const double num = ax * crx + ay * cry + az * crz;
  const double abc = la * lb * lc;
  const double den = abc + (ax * bx + ay * by + az * bz) * lc + (bx * cx + by * cy + bz * cz) * la +
                     (cx * ax + cy * ay + cz * az) * lb;
  if (fabs(num) < guard * abc && den <= 0.0) {  // coplanar, inside the rim (:408)
    acc.on = true;
    return;
  }
  cmul_track(acc.st, den, num);
  if ((++acc.n & 7) == 0) renorm(acc.st);
}

__global__ void __launch_bounds__(kSaBlock)
k_solid_angle(const double* __restrict__ P, int64_t nP, const double* __restrict__ tri,
              int64_t nT, double guard, double* __restrict__ out, int8_t* __restrict__ on) {
  __shared__ double sT[9][kTileT];
  const int64_t q0 = ((int64_t)blockIdx.x * kSaBlock + threadIdx.x) * 2;
  double p[2][3];
  SaAcc acc[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int64_t q = q0 + j < nP ? q0 + j : nP - 1;
    for (int k = 0; k < 3; ++k) p[j][k] = P[3 * q + k];
    acc[j].st.Zr = 1.0;
    acc[j].st.Zi = 0.0;
    acc[j].st.wraps = 0;
    acc[j].n = 0;
    acc[j].on = false;
  }
  const double guard2 = guard * guard;
  for (int64_t f0 = 0; f0 < nT; f0 += kTileT) {
    const int nt = (int)min((int64_t)kTileT, nT - f0);
    __syncthreads();
    for (int k = threadIdx.x; k < 9 * nt; k += kSaBlock) {
      const int c = k / nt, f = k - c * nt;
      sT[c][f] = tri[(int64_t)c * nT + f0 + f];
    }
    __syncthreads();
    for (int f = 0; f < nt; ++f) {
      double t[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) t[c] = sT[c][f];
#pragma unroll
      for (int j = 0; j < 2; ++j) sa_term(acc[j], p[j][0], p[j][1], p[j][2], t, guard2, guard);
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (q0 + j >= nP) continue;
    out[q0 + j] = 2.0 * seg_angle(acc[j].st);
    on[q0 + j] = acc[j].on ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// ray / triangle-mesh all hits
// ---------------------------------------------------------------------------

struct TriBvhDev {
  const double *node_min, *node_max;
  const int64_t *node_left, *node_right, *node_start, *node_count, *tri_order;
  int64_t n_nodes;
  const double *V0, *E1, *E2, *NN, *NH, *C, *R2;
  int64_t n_tris;
};

struct TriHit {
  double t, dd, u, v;
  int64_t tri;
  int par;
};

// _ray_tris_hits_numpy (:312-363) for one triangle; returns 1 on a hit
__device__ __forceinline__ int tri_hit(const TriBvhDev& b, int64_t f, const double o[3],
                                       const double d[3], double t_lo, double t_hi,
                                       double tang_eps, double plane_tol, TriHit& h) {
  const double* v0 = b.V0 + 3 * f;
  const double* e1 = b.E1 + 3 * f;
  const double* e2 = b.E2 + 3 * f;
  const double hx = d[1] * e2[2] - d[2] * e2[1], hy = d[2] * e2[0] - d[0] * e2[2],
               hz = d[0] * e2[1] - d[1] * e2[0];
  const double a = e1[0] * hx + e1[1] * hy + e1[2] * hz;
  const double nn = b.NN[f];
  const double sx = o[0] - v0[0], sy = o[1] - v0[1], sz = o[2] - v0[2];
  if (fabs(a) <= tang_eps * nn) {
    // parallel: tangent contact if the line lies in the plane near the triangle
    const double* nh = b.NH + 3 * f;
    const double pdist = fabs(sx * nh[0] + sy * nh[1] + sz * nh[2]);
    const double* c = b.C + 3 * f;
    const double tcx = c[0] - o[0], tcy = c[1] - o[1], tcz = c[2] - o[2];
    const double tca = tcx * d[0] + tcy * d[1] + tcz * d[2];
    const double d2 = tcx * tcx + tcy * tcy + tcz * tcz - tca * tca;
    if (pdist <= plane_tol && d2 <= b.R2[f] && tca >= t_lo && tca <= t_hi) {
      h.t = tca;
      h.dd = 0.0;
      h.u = h.v = 1.0 / 3.0;
      h.tri = f;
      h.par = 1;
      return 1;
    }
    return 0;
  }
  const double inv = 1.0 / a;
  const double u = inv * (sx * hx + sy * hy + sz * hz);
  const double qx = sy * e1[2] - sz * e1[1], qy = sz * e1[0] - sx * e1[2],
               qz = sx * e1[1] - sy * e1[0];
  const double v = inv * (qx * d[0] + qy * d[1] + qz * d[2]);
  const double t = inv * (e2[0] * qx + e2[1] * qy + e2[2] * qz);
  if (u >= -1e-12 && u <= 1.0 + 1e-12 && v >= -1e-12 && u + v <= 1.0 + 1e-12 && t >= t_lo &&
      t <= t_hi) {
    h.t = t;
    h.dd = -a / nn;
    h.u = u;
    h.v = v;
    h.tri = f;
    h.par = 0;
    return 1;
  }
  return 0;
}

// slab test of a BVH node, widened so it never culls what brute force finds
__device__ __forceinline__ bool node_slab(const TriBvhDev& b, int64_t node, const double o[3],
                                          const double d[3], double t_lo, double t_hi,
                                          double pad) {
  double tmin = t_lo, tmax = t_hi;
  for (int k = 0; k < 3; ++k) {
    const double lo = b.node_min[3 * node + k] - pad, hi = b.node_max[3 * node + k] + pad;
    if (d[k] == 0.0) {
      if (o[k] < lo || o[k] > hi) return false;
    } else {
      const double inv = 1.0 / d[k];
      double t0 = (lo - o[k]) * inv, t1 = (hi - o[k]) * inv;
      if (t0 > t1) {
        const double x = t0;
        t0 = t1;
        t1 = x;
      }
      tmin = fmax(tmin, t0 - 1e-9 * (1.0 + fabs(t0)));
      tmax = fmin(tmax, t1 + 1e-9 * (1.0 + fabs(t1)));
      if (tmax < tmin) return false;
    }
  }
  return true;
}

constexpr int kBvhStack = 128;  // as the reference (:258)

// kFill = false: count hits per ray; true: write them at offs[r]
template <bool kFill>
__global__ void k_ray_tris(TriBvhDev b, const double* __restrict__ org,
                           const double* __restrict__ dir, int64_t R, double t_lo, double t_hi,
                           double tang_eps, double plane_tol, double pad,
                           int64_t* __restrict__ counts, const int64_t* __restrict__ offs,
                           double* __restrict__ ts, int64_t* __restrict__ tris,
                           double* __restrict__ dd, double* __restrict__ us,
                           double* __restrict__ vs, unsigned long long* __restrict__ keys,
                           int* __restrict__ overflow) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double o[3] = {org[3 * r], org[3 * r + 1], org[3 * r + 2]};
  const double d[3] = {dir[3 * r], dir[3 * r + 1], dir[3 * r + 2]};
  int64_t n = 0;
  const int64_t base = kFill ? offs[r] : 0;
  int64_t stack[kBvhStack];
  int top = 0;
  if (b.n_nodes > 0) stack[top++] = 0;
  while (top > 0) {
    const int64_t node = stack[--top];
    if (!node_slab(b, node, o, d, t_lo, t_hi, pad)) continue;
    if (b.node_left[node] < 0) {
      const int64_t s0 = b.node_start[node], s1 = s0 + b.node_count[node];
      for (int64_t k = s0; k < s1; ++k) {
        TriHit h;
        if (!tri_hit(b, b.tri_order[k], o, d, t_lo, t_hi, tang_eps, plane_tol, h)) continue;
        if (kFill) {
          const int64_t i = base + n;
          ts[i] = h.t;
          tris[i] = h.tri;
          dd[i] = h.dd;
          us[i] = h.u;
          vs[i] = h.v;
          // (ray, kind, triangle): the numpy twin's order within a ray
          keys[i] = ((unsigned long long)r * 2ull + (unsigned long long)h.par) *
                        (unsigned long long)b.n_tris +
                    (unsigned long long)h.tri;
        }
        ++n;
      }
    } else if (top + 2 <= kBvhStack) {
      stack[top++] = b.node_left[node];
      stack[top++] = b.node_right[node];
    } else {
      *overflow = 1;
    }
  }
  if (!kFill) counts[r] = n;
}

template <class T>
__global__ void k_gather_perm(int64_t n, const int64_t* __restrict__ perm, const T* __restrict__ src,
                              T* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

__global__ void k_iota(int64_t n, int64_t* __restrict__ x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}

// device buffers freed on scope exit (host-synchronous entry points)
struct DevBufs {
  std::vector<void*> p;
  cudaError_t err = cudaSuccess;
  template <class T>
  T* get(size_t n) {
    void* x = nullptr;
    if (err != cudaSuccess) return nullptr;
    err = cudaMalloc(&x, n * sizeof(T) + 16);
    if (err == cudaSuccess) p.push_back(x);
    return (T*)x;
  }
  template <class T>
  T* up(const T* h, size_t n) {
    T* d = get<T>(n);
    if (d && n) err = cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice);
    return d;
  }
  ~DevBufs() {
    for (void* x : p) cudaFree(x);
  }
};

// sort 64-bit keys, returning the permutation (values = original index)
static cudaError_t sort_keys(DevBufs& db, unsigned long long* keys, int64_t n, int end_bit,
                             unsigned long long** keys_out, int64_t** perm_out) {
  unsigned long long* k2 = db.get<unsigned long long>(n);
  int64_t* v1 = db.get<int64_t>(n);
  int64_t* v2 = db.get<int64_t>(n);
  if (db.err != cudaSuccess) return db.err;
  k_iota<<<(unsigned)((n + 255) / 256), 256>>>(n, v1);
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, k2, v1, v2, (int)n, 0, end_bit);
  if (e != cudaSuccess) return e;
  void* tmp = db.get<char>(tb);
  if (db.err != cudaSuccess) return db.err;
  e = cub::DeviceRadixSort::SortPairs(tmp, tb, keys, k2, v1, v2, (int)n, 0, end_bit);
  *keys_out = k2;
  *perm_out = v2;
  return e;
}

static int bits_for(unsigned long long x) {
  int b = 1;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

}  // namespace gwn

using namespace gwn;

#define CKM(call)                                                             \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      set_error("%s failed: %s", #call, cudaGetErrorString(e_));             \
      return (e_ == cudaErrorMemoryAllocation) ? GWN_E_OOM : GWN_E_CUDA;      \
    }                                                                         \
  } while (0)

extern "C" int gwn_solid_angle_many(const double* V, int64_t nV, const int64_t* T, int64_t nT,
                                    const double* P, int64_t nP, double guard, double* out,
                                    int8_t* on_surface, int device) {
  if (nV < 0 || nT < 0 || nP < 0 || (nP > 0 && (!P || !out || !on_surface)) ||
      (nT > 0 && (!V || !T))) {
    set_error("gwn_solid_angle_many: invalid arguments");
    return GWN_E_INVALID;
  }
  if (nP == 0) return GWN_OK;
  CKM(cudaSetDevice(device));
  DevBufs db;
  const double* dP = db.up(P, 3 * (size_t)nP);
  double* dout = db.get<double>(nP);
  int8_t* don = db.get<int8_t>(nP);
  double* tri = db.get<double>(9 * (size_t)(nT > 0 ? nT : 1));
  int* bad = db.get<int>(1);
  CKM(db.err);
  CKM(cudaMemset(bad, 0, sizeof(int)));
  if (nT > 0) {
    const double* dV = db.up(V, 3 * (size_t)nV);
    const int64_t* dT = db.up(T, 3 * (size_t)nT);
    CKM(db.err);
    k_tri_gather<<<(unsigned)((nT + 255) / 256), 256>>>(dV, dT, nT, nV, tri, bad);
    CKM(cudaGetLastError());
  }
  const unsigned blocks = (unsigned)((nP + 2 * kSaBlock - 1) / (2 * kSaBlock));
  k_solid_angle<<<blocks, kSaBlock>>>(dP, nP, tri, nT, guard, dout, don);
  CKM(cudaGetLastError());
  int hbad = 0;
  CKM(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (hbad) {
    set_error("gwn_solid_angle_many: triangle index out of range");
    return GWN_E_INVALID;
  }
  CKM(cudaMemcpy(out, dout, sizeof(double) * nP, cudaMemcpyDeviceToHost));
  CKM(cudaMemcpy(on_surface, don, nP, cudaMemcpyDeviceToHost));
  return GWN_OK;
}

extern "C" int64_t gwn_ray_tris_hits(const gwn_tri_bvh* bvh, const double* origins,
                                     const double* dirs, int64_t R, double t_lo, double t_hi,
                                     double tang_eps, double plane_tol, int64_t* offs,
                                     double* ts, int64_t* tris, double* dotdn, double* us,
                                     double* vs, int64_t cap, int device) {
  if (!bvh || R < 0 || (R > 0 && (!origins || !dirs || !offs)) || bvh->n_tris < 0 ||
      bvh->n_nodes < 0) {
    set_error("gwn_ray_tris_hits: invalid arguments");
    return GWN_E_INVALID;
  }
  if (R == 0) {
    if (offs) offs[0] = 0;
    return 0;
  }
  CKM(cudaSetDevice(device));
  DevBufs db;
  const int64_t F = bvh->n_tris, N = bvh->n_nodes;
  TriBvhDev b;
  b.n_nodes = F > 0 ? N : 0;
  b.n_tris = F > 0 ? F : 1;
  b.node_min = db.up(bvh->node_min, 3 * (size_t)N);
  b.node_max = db.up(bvh->node_max, 3 * (size_t)N);
  b.node_left = db.up(bvh->node_left, (size_t)N);
  b.node_right = db.up(bvh->node_right, (size_t)N);
  b.node_start = db.up(bvh->node_start, (size_t)N);
  b.node_count = db.up(bvh->node_count, (size_t)N);
  b.tri_order = db.up(bvh->tri_order, (size_t)F);
  b.V0 = db.up(bvh->V0, 3 * (size_t)F);
  b.E1 = db.up(bvh->E1, 3 * (size_t)F);
  b.E2 = db.up(bvh->E2, 3 * (size_t)F);
  b.NN = db.up(bvh->NN, (size_t)F);
  b.NH = db.up(bvh->NH, 3 * (size_t)F);
  b.C = db.up(bvh->C, 3 * (size_t)F);
  b.R2 = db.up(bvh->R2, (size_t)F);
  const double* dO = db.up(origins, 3 * (size_t)R);
  const double* dD = db.up(dirs, 3 * (size_t)R);
  int64_t* cnt = db.get<int64_t>(R + 1);
  int64_t* doffs = db.get<int64_t>(R + 1);
  int* ovf = db.get<int>(1);
  CKM(db.err);
  CKM(cudaMemset(ovf, 0, sizeof(int)));
  CKM(cudaMemset(cnt + R, 0, sizeof(int64_t)));
  // slab widening: the largest circumradius (a parallel-ray tangent contact
  // only needs the line within R of the centroid, :349-356, which the
  // triangle's own box need not contain) plus a relative 1e-9 of the extent
  double pad = 0.0;
  if (N > 0) {
    double ext = 0.0, r2max = 0.0;
    for (int k = 0; k < 3; ++k)
      ext = fmax(ext, fmax(fabs(bvh->node_min[k]), fabs(bvh->node_max[k])));
    for (int64_t f = 0; f < F; ++f) r2max = fmax(r2max, bvh->R2[f]);
    pad = sqrt(r2max) + 1e-9 * (1.0 + ext);
  }
  const unsigned g = (unsigned)((R + 127) / 128);
  k_ray_tris<false><<<g, 128>>>(b, dO, dD, R, t_lo, t_hi, tang_eps, plane_tol, pad, cnt, nullptr,
                                nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ovf);
  CKM(cudaGetLastError());
  size_t tb = 0;
  CKM(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, doffs, (int)(R + 1)));
  void* tmp = db.get<char>(tb);
  CKM(db.err);
  CKM(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, doffs, (int)(R + 1)));
  int hovf = 0;
  CKM(cudaMemcpy(&hovf, ovf, sizeof(int), cudaMemcpyDeviceToHost));
  if (hovf) {
    set_error("gwn_ray_tris_hits: BVH deeper than the traversal stack");
    return GWN_E_INVALID;
  }
  CKM(cudaMemcpy(offs, doffs, sizeof(int64_t) * (R + 1), cudaMemcpyDeviceToHost));
  const int64_t total = offs[R];
  if (total > cap || total == 0) return total;
  if (!ts || !tris || !dotdn || !us || !vs) {
    set_error("gwn_ray_tris_hits: null output buffers");
    return GWN_E_INVALID;
  }
  double* t1 = db.get<double>(total);
  double* d1 = db.get<double>(total);
  double* u1 = db.get<double>(total);
  double* v1 = db.get<double>(total);
  int64_t* f1 = db.get<int64_t>(total);
  unsigned long long* key = db.get<unsigned long long>(total);
  CKM(db.err);
  k_ray_tris<true><<<g, 128>>>(b, dO, dD, R, t_lo, t_hi, tang_eps, plane_tol, pad, nullptr, doffs,
                               t1, f1, d1, u1, v1, key, ovf);
  CKM(cudaGetLastError());
  unsigned long long* ks = nullptr;
  int64_t* perm = nullptr;
  const int end_bit = bits_for((unsigned long long)R * 2ull * (unsigned long long)b.n_tris);
  CKM(sort_keys(db, key, total, end_bit, &ks, &perm));
  double* t2 = db.get<double>(total);
  double* d2 = db.get<double>(total);
  double* u2 = db.get<double>(total);
  double* v2 = db.get<double>(total);
  int64_t* f2 = db.get<int64_t>(total);
  CKM(db.err);
  const unsigned gt = (unsigned)((total + 255) / 256);
  k_gather_perm<double><<<gt, 256>>>(total, perm, t1, t2);
  k_gather_perm<double><<<gt, 256>>>(total, perm, d1, d2);
  k_gather_perm<double><<<gt, 256>>>(total, perm, u1, u2);
  k_gather_perm<double><<<gt, 256>>>(total, perm, v1, v2);
  k_gather_perm<int64_t><<<gt, 256>>>(total, perm, f1, f2);
  CKM(cudaGetLastError());
  CKM(cudaMemcpy(ts, t2, sizeof(double) * total, cudaMemcpyDeviceToHost));
  CKM(cudaMemcpy(dotdn, d2, sizeof(double) * total, cudaMemcpyDeviceToHost));
  CKM(cudaMemcpy(us, u2, sizeof(double) * total, cudaMemcpyDeviceToHost));
  CKM(cudaMemcpy(vs, v2, sizeof(double) * total, cudaMemcpyDeviceToHost));
  CKM(cudaMemcpy(tris, f2, sizeof(int64_t) * total, cudaMemcpyDeviceToHost));
  return total;
}
