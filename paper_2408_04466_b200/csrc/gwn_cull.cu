// gwn_cull.cu -- K2: query x patch cull by 2-D LBVH traversal in the ray
// frame of the round.
//
// Replaces the reference's per-(ray, patch) `patch.aabb()` + ray_aabb_clip
// (surfaces.py:636-639, geometry.py:198-219): with every ray of the round
// parallel to d, a leaf sub-patch can be hit only if the query's projection
// (p.e1, p.e2) lies in the leaf's projected control box and the leaf reaches
// past p along d (cmax >= p.d).  Two passes with the same deterministic
// traversal: count, (scan), fill -> (query slot, leaf) candidates grouped by
// query slot.
#include "gwn_internal.h"

namespace gwn {

constexpr int kStack = 64;  // >= LBVH depth bound (30-bit Morton + 32-bit index tie-break)

template <bool kFill>
__device__ __forceinline__ int traverse(const Node* __restrict__ nodes,
                                        const double* __restrict__ leafbox, int64_t P,
                                        double qa, double qb, double qc, int32_t slot,
                                        int32_t* __restrict__ out_slot,
                                        int32_t* __restrict__ out_patch) {
  int count = 0;
  if (P == 1) {
    const double* b = leafbox;
    if (qa >= b[0] && qa <= b[1] && qb >= b[2] && qb <= b[3] && b[4] >= qc) {
      if (kFill) { out_slot[0] = slot; out_patch[0] = 0; }
      count = 1;
    }
    return count;
  }
  int stack[kStack];
  int top = 0;
  int node = 0;
  for (;;) {
    const Node& n = nodes[node];
    int next = -1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      bool hit = qa >= n.alo[c] && qa <= n.ahi[c] && qb >= n.blo[c] && qb <= n.bhi[c] &&
                 n.cmax[c] >= qc;
      if (!hit) continue;
      int ch = n.child[c];
      if (ch < 0) {
        if (kFill) {
          out_slot[count] = slot;
          out_patch[count] = ~ch;
        }
        ++count;
      } else if (next < 0) {
        next = ch;
      } else if (top < kStack) {
        stack[top++] = ch;
      }
    }
    if (next >= 0) {
      node = next;
    } else if (top > 0) {
      node = stack[--top];
    } else {
      break;
    }
  }
  return count;
}

__device__ __forceinline__ void query_proj(const Frame& f, const double* __restrict__ pos,
                                           int32_t q, double& qa, double& qb, double& qc) {
  double x = pos[3 * (int64_t)q], y = pos[3 * (int64_t)q + 1], z = pos[3 * (int64_t)q + 2];
  qa = x * f.e1[0] + y * f.e1[1] + z * f.e1[2];
  qb = x * f.e2[0] + y * f.e2[1] + z * f.e2[2];
  qc = x * f.d[0] + y * f.d[1] + z * f.d[2];
}

__global__ void k_cull_count(const Node* __restrict__ nodes, const double* __restrict__ leafbox,
                             int64_t P, Frame f, int32_t m, const int32_t* __restrict__ active,
                             const double* __restrict__ pos, int64_t* __restrict__ counts,
                             double* __restrict__ qproj) {
  int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  int32_t q = active ? active[s] : s;
  double qa, qb, qc;
  query_proj(f, pos, q, qa, qb, qc);
  qproj[3 * (int64_t)s] = qa;
  qproj[3 * (int64_t)s + 1] = qb;
  qproj[3 * (int64_t)s + 2] = qc;
  counts[s] = traverse<false>(nodes, leafbox, P, qa, qb, qc, s, nullptr, nullptr);
}

__global__ void k_cull_fill(const Node* __restrict__ nodes, const double* __restrict__ leafbox,
                            int64_t P, Frame f, int32_t m, const int32_t* __restrict__ active,
                            const double* __restrict__ pos, const int64_t* __restrict__ offs,
                            int32_t* __restrict__ pair_slot, int32_t* __restrict__ pair_patch) {
  int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  int32_t q = active ? active[s] : s;
  double qa, qb, qc;
  query_proj(f, pos, q, qa, qb, qc);
  int64_t o = offs[s];
  traverse<true>(nodes, leafbox, P, qa, qb, qc, s, pair_slot + o, pair_patch + o);
}

cudaError_t launch_cull_count(const gwn_scene* sc, const Round& rd, int32_t m,
                              const int32_t* active, const double* pos, int64_t* counts,
                              double* qproj, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_cull_count<<<(m + 127) / 128, 128, 0, st>>>(rd.nodes, rd.leafbox, rd.n_leaves, rd.f, m, active,
                                                pos, counts, qproj);
  return cudaGetLastError();
}

cudaError_t launch_cull_fill(const gwn_scene* sc, const Round& rd, int32_t m,
                             const int32_t* active, const double* pos, const int64_t* offs,
                             int32_t* pair_slot, int32_t* pair_patch, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_cull_fill<<<(m + 127) / 128, 128, 0, st>>>(rd.nodes, rd.leafbox, rd.n_leaves, rd.f, m, active, pos,
                                               offs, pair_slot, pair_patch);
  return cudaGetLastError();
}

}  // namespace gwn
