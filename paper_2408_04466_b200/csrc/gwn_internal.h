// gwn_internal.h -- host/device shared definitions of libgwn_b200.so.
//
// Data layout in HBM:
//   ctrl      (P,16,3) f64   original control nets, i = u index (row-major)
//   proj[r]   (P,48)   f64   per direction round r: the 16 control points in
//                            the ray frame (e1,e2,d): [A0..A15 | B0..B15 | C0..C15]
//   nodes[r]  (P-1)    Node  2-D LBVH over the projected control hulls; each
//                            internal node stores both children's boxes
//   verts     (V,3)    f64   SoA x|y|z of the net boundary polylines, S per edge
#pragma once

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#include <array>
#include <mutex>
#include <utility>
#include <deque>
#include <vector>

#include "../../include/gwn_b200.h"

namespace gwn {

// per-query flag bits accumulated over a round
enum : int32_t {
  FLAG_RESHOOT = 1,   // tangency / grazing / ambiguous root set -> new direction
  FLAG_BAND = 2,      // ray within the polyline/curve band of a net segment
  FLAG_ONSURF = 4,    // a hit with |t| <= on_surface_t -> jitter
  FLAG_DEGEN = 8,     // query on a boundary vertex -> jitter
  FLAG_OVERFLOW = 16, // all_hits: root set larger than the record buffer
};

// device counters (index into a u64 array)
enum : int {
  CNT_CANDIDATES = 0,
  CNT_NODES = 1,
  CNT_NEWTON = 2,
  CNT_ROOTS = 3,
  CNT_SEGMENTS = 4,
  CNT_MAXNODES = 5,  // max DFS nodes of one fallback item (diagnostic)
  CNT_BIGITEMS = 6,  // slowest fallback warp: cycles<<24 | tree levels<<16 | code levels<<8 | items
  CNT_MAXLEVELS = 7, // deepest fallback BFS, in levels (diagnostic)
  CNT_FAR = 8,       // (query, entry) pairs taken by the far-field expansion
  CNT_FAR_TERMS = 9, // solid-harmonic terms those expansions summed
  CNT_NEAR = 10,     // (query, entry) pairs summed exactly (far-field scenes)
  CNT_LOCAL = 11,    // queries whose far field came from a leaf's local expansion
  CNT_SHADOW = 12,   // far pairs whose forward half-line crosses the cycle's sphere
  CNT_N = 13,
};

struct Frame {
  double e1[3], e2[3], d[3];
};

// one ray-patch root in record mode (ray reuse): slot, sign, t
struct HitRec {
  int32_t slot;
  int32_t sign;
  double t;
};

struct RecordSink {
  HitRec* rec;
  unsigned long long* count;
  unsigned long long cap;
};

struct DevParams {
  double residual, dedup, tangent, edge_graze, degenerate;
  double domain_tol, t_tol, on_surface_t, band_factor;
};

// 2-D LBVH node in the ray frame.  Child c's box: a in [alo,ahi], b in
// [blo,bhi], patch extent along d up to cmax.  child >= 0: internal node,
// child < 0: leaf patch ~child.
struct alignas(16) Node {
  double alo[2], ahi[2], blo[2], bhi[2], cmax[2];
  int32_t child[2];
};

struct LeafRec;

// Local expansions of the boundary term's far field for one round
// (gwn_fmm.cu): an octree over the scene cube; every (box, closed cycle)
// pair accepted at the coarsest level whose error bound and line test hold
// is translated (M2L) into the box's local expansion, pushed down (L2L) to
// the leaves.  Per leaf: its local coefficients and the list of entries left
// to the per-query path (the "leftover" list).
struct FmmRound {
  int L = 0;                    // leaf level
  int64_t n_leaf = 0;           // 8^L leaf boxes, row-major (ix, iy, iz)
  double2* leafL = nullptr;     // (n_leaf, kFmmLT) local coefficients L_j^k, k >= 0
  int32_t* loff = nullptr;      // (n_leaf + 2) leftover list offsets; list n_leaf = every entry
  int32_t* lent = nullptr;      // leftover entries, ascending per list
  int64_t m2l_pairs = 0;        // (box, cycle) translations
  int64_t leftover = 0;         // total leftover entries over the leaves
  double ms_build = 0.0;
};

// packed uniform-grid entry: a leaf's cull box rounded outward to float
struct CellEnt {
  float alo, ahi, blo, bhi, cmax;
  int32_t leaf;
};

struct Round {
  Frame f;
  double* proj = nullptr;      // (P,48)
  double* powc = nullptr;      // (P,48) proj in the power basis (K3 Newton, Horner)
  int64_t n_leaves = 0;
  LeafRec* leaves = nullptr;   // (n_leaves) adaptive leaf sub-patches
  double* leafbox = nullptr;   // (n_leaves,5) cull boxes: a lo/hi, b lo/hi, c max
  Node* nodes = nullptr;       // (n_leaves-1) LBVH over the leaf boxes
  double amin = 0, ainv = 0, bmin = 0, binv = 0;  // projected scene box (Morton keys)
  double* vproj = nullptr;     // (3,V) boundary vertices in the ray frame (K4)
  double* ffg = nullptr;       // (ff_n,3) far-field cycle centres in the ray frame
  double* ffa = nullptr;       // (ff_n,6) sliver chord end points in the ray frame
  int8_t* ffw = nullptr;       // (ff_n,kWG,kWG) shadow winding grids (k_ff_wind)
  double* ffwg = nullptr;      // (ff_n,3) grid origin (X, Y) and inverse cell size
  // uniform grid over the leaf boxes (K2 point location); used when its
  // cells stay short, else the LBVH
  bool use_grid = false;
  int32_t ga = 0, gb = 0;      // cells along a, b
  double gx0 = 0, gy0 = 0, gia = 0, gib = 0;  // origin and inverse cell size
  int32_t* cell_offs = nullptr;    // (ga*gb+1) exclusive offsets
  CellEnt* cell_ent = nullptr;     // packed leaf boxes per cell
  int64_t grid_entries = 0;
  // fold trees of the uncertified leaves (k_foldtree): the tree of leaf i
  // is nodes [sub_offs[i], sub_offs[i+1]) in preorder, node k's subtree is
  // [k, k + subskip[k]) (1 = leaf); boxes as leafbox
  LeafRec* sub = nullptr;
  double* subbox = nullptr;
  int32_t* subskip = nullptr;
  int4* subgc = nullptr;        // grandchild offsets (k_foldtree_gc), -1 = none
  int64_t* sub_offs = nullptr;  // (n_leaves+1), null when no leaf needed it
  int64_t n_sub = 0;
  int sub_level = 0;
  // far-field local expansions (built on first use by a large eval; null = per-pair path)
  FmmRound* fmm = nullptr;
};

}  // namespace gwn

struct gwn_scene {
  gwn_params prm;
  gwn::DevParams dprm;
  int device = 0;
  int sm_count = 0;
  int64_t P = 0;
  double bbox_min[3], bbox_max[3], diag = 0.0;
  double* ctrl = nullptr;       // device (P,48)
  // net boundary
  int64_t n_edges = 0;          // after expanding multiplicities
  int32_t S = 0;
  double* verts = nullptr;      // (3,V) SoA, V = n_edges*S
  double* band_h = nullptr;     // (n_edges)
  // far field of the boundary term (gwn_farfield.cu): the net edges are
  // grouped into entries (closed cycles, slivers, exact-only pieces), each a
  // contiguous edge range; ff_n = 0 when off
  int32_t ff_n = 0;             // entries
  int32_t ff_expanded = 0;      // entries with a multipole expansion
  int32_t* ff_eoff = nullptr;   // (ff_n+1) edge range of each entry
  double* ff_g = nullptr;       // (ff_n,3) entry centre (world)
  double* ff_r = nullptr;       // (ff_n,2) R_min^2 (+inf: exact only), line radius^2
  double* ff_D = nullptr;       // (ff_n, kFFTerms, 2) double-layer moments
  double* ff_lv = nullptr;      // (ff_n, kFFLevels) R^2 thresholds of the adaptive orders
  double ff_tau = 0.0;          // per-entry truncation bound (Omega units, kFFDw budget)
  int32_t* ff_chord = nullptr;  // (ff_n) sliver entries: edge of the closing chord, else -1
  std::vector<double> ff_chord_host;  // (ff_n,6) chord start / end (world), zeros for cycles
  // octree of the far field's local expansions (gwn_fmm.cu): cube, leaf level
  // (0 = off) and, per (entry, level), the distance from a box centre beyond
  // which the entry's translation into that box meets the error budget
  // (+inf: never -- slivers and exact-only entries)
  int fmm_L = 0;
  double fmm_x0[3] = {0, 0, 0}, fmm_side = 0.0;
  double* fmm_dmin = nullptr;   // (ff_n, fmm_L + 1)
  std::vector<double> ff_g_host;
  // per-round caches
  std::mutex mu;
  // deques: push_back never moves existing rounds, so a Round* taken under
  // `mu` stays valid while other threads add rounds
  std::deque<gwn::Round> rounds;
  // candidate (query, leaf) pairs per query seen so far (buffer sizing)
  double pairs_per_query = 4.0;
  // rounds for explicit ray directions (ray reuse), keyed by direction
  std::deque<std::pair<std::array<double, 3>, gwn::Round>> dir_rounds;
  // last-eval stats
  gwn_stats stats;
  int timed = 0;
};

namespace gwn {

// GPU-side timeline (GWN_TIMELINE=1, development aid): timing events
// recorded between the ops of one eval on whichever stream runs them;
// recording an event does not order the streams.
struct GpuTimeline {
  cudaEvent_t ev[48];
  const char* name[48];
  int n = 0;
  void mark(cudaStream_t s, const char* nm) {
    if (n >= 48 || cudaEventCreate(&ev[n]) != cudaSuccess) return;
    cudaEventRecord(ev[n], s);
    name[n++] = nm;
  }
  void dump() {
    for (int k = 0; k < n; ++k) {
      float ms = 0.f;
      const cudaError_t e = cudaEventElapsedTime(&ms, ev[0], ev[k]);
      fprintf(stderr, "[gwn-tl] %-26s %9.1f us %s\n", name[k], ms * 1e3f,
              e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    for (int k = 0; k < n; ++k) cudaEventDestroy(ev[k]);
    n = 0;
  }
};
extern thread_local GpuTimeline* g_tl;
inline void tl_mark(cudaStream_t s, const char* nm) {
  if (g_tl) g_tl->mark(s, nm);
}

struct K3Queues;  // gwn_k3.cuh

// per-slot accumulators the cull kernel zeroes for its round (nullable)
struct CullZero {
  int32_t* chi = nullptr;
  int32_t* flags = nullptr;
};

// launchers (stream-ordered); defined in the .cu files
cudaError_t build_round(gwn_scene* sc, int r, cudaStream_t st);            // gwn_bvh.cu
cudaError_t build_round_dir(gwn_scene* sc, const double d[3], Round& rd, cudaStream_t st);
void free_round(Round& rd);
cudaError_t launch_cull(const gwn_scene* sc, const Round& rd, int32_t m, const int32_t* active,
                        const double* pos, double* qproj, unsigned long long* pair_count,
                        int64_t cap, CullZero z, const K3Queues& Q, unsigned long long* counters,
                        cudaStream_t st);  // gwn_cull.cu: K2 -> Q.pairs                                     // gwn_cull.cu
cudaError_t launch_intersect(const gwn_scene* sc, const Round& rd, const K3Queues& Q,
                             const unsigned long long* npairs_dev, const double* qproj,
                             int32_t* chi, int32_t* flags, unsigned long long* counters,
                             unsigned long long* newton_work, cudaEvent_t* ev4,
                             cudaEvent_t* join, const RecordSink* rec,
                             cudaStream_t st);  // gwn_wavefront.cu: candidates, fallback, Newton
// K3 queues in `scratch` (intersect_scratch_bytes(cap)); k3cnt: 4 zeroed
// device counters per round ([0] fallback items, [1] Newton items,
// [2] overflow, [3] Newton work)
// P > kTabMaxP adds the patch bins of the Newton pass (K3Queues::nkey ...);
// rounds of fewer than kBinMinQueries queries pass P = 0 (no bins).
constexpr int32_t kBinMinQueries = 1 << 16;
K3Queues k3_queues(void* scratch, int64_t cap, unsigned long long* k3cnt, int64_t P);
size_t intersect_scratch_bytes(int64_t pair_cap, int64_t P);
cudaError_t launch_boundary(const gwn_scene* sc, const Round& rd, int32_t m,
                            const int32_t* active, const double* pos, double* bpart, int nchunk,
                            int32_t* flags, unsigned long long* counters, cudaStream_t st,
                            const int32_t* order = nullptr,
                            cudaEvent_t* evb = nullptr);                      // gwn_boundary.cu
int boundary_chunks(const gwn_scene* sc, int32_t m);  // partial rows (exact chunks + far row)
cudaError_t build_farfield(gwn_scene* sc, const double* ectrl);     // gwn_farfield.cu
cudaError_t ff_init_constants();                                   // gwn_boundary.cu
void free_farfield(gwn_scene* sc);
cudaError_t launch_ff_order(const gwn_scene* sc, int32_t m, const int32_t* active,
                            const double* pos, void* scratch, int32_t* order, cudaStream_t st);
size_t ff_order_scratch_bytes(int32_t m);
cudaError_t launch_column_order(const Round& rd, int32_t m, const double* pos, void* scratch,
                                int32_t* order, cudaStream_t st);  // gwn_farfield.cu
cudaError_t launch_vproj(const gwn_scene* sc, Round& rd, cudaStream_t st);  // gwn_boundary.cu
// far-field local expansions (gwn_fmm.cu): scene-level acceptance table,
// per-round octree build (caller holds sc->mu), release
cudaError_t fmm_setup_scene(gwn_scene* sc, const std::vector<double>& rho,
                            const std::vector<double>& aabs, const std::vector<char>& closed);
cudaError_t build_fmm_round(const gwn_scene* sc, Round& rd, cudaStream_t st);
void free_fmm_round(Round& rd);
cudaError_t selftest_rsqrt(int64_t n, unsigned long long* max_ulp_host);
cudaError_t launch_all_hits(const Round& rd, const DevParams& prm, const double* o, double t_lo,
                            double t_hi, double* out, int32_t* count, int32_t cap,
                            cudaStream_t st);
cudaError_t launch_single_loop(const double* loop, int64_t B, const double* o, const double* d,
                               const double* hit_ts, const int64_t* hit_signs, int64_t H,
                               const double* qts, int64_t K, double t_eps, double deg, double* w,
                               int8_t* ok, cudaStream_t st);

// the engine body shared by gwn_eval and the ray-reuse fallback (gwn_engine.cu):
// device buffers; qidx (nullable, device) gives the global id of each query
int eval_impl(gwn_scene* sc, const double* d_q, int64_t n, int64_t index_base,
              const int64_t* qidx, double* d_w, int8_t* d_st, cudaStream_t st, gwn_stats& stats);

// host helpers (gwn_scene.cu)
void make_frame(const double d[3], Frame* f);
void set_error(const char* fmt, ...);

}  // namespace gwn
