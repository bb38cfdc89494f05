/* include/gwn_b200.h -- C ABI of libgwn_b200.so (B200 / sm_100a).
 *
 * Batched generalized winding numbers of query points against bicubic
 * Bezier patches (arXiv 2408.04466).  Plain pointers and sizes only; no
 * torch types.  Each entry point replaces a reference interface:
 *
 *   gwn_scene_create   SPEC.md:355-365 `Scene` construction (patches +
 *                      aggregated boundary loops, surfaces.py:611-626) and the
 *                      per-patch `aabb()` of surfaces.py:562-564 / 636
 *   gwn_eval           SPEC.md:371-380 engine.winding_number, batched; the
 *                      per-query sum over patch.all_hits (surfaces.py:634-701)
 *                      and the boundary term (_kernels.py:723-798), with the
 *                      jitter/re-shoot policy of SPEC.md:320,373-375,427
 *   gwn_all_hits       patch.all_hits(ray) (surfaces.py:587-589 protocol,
 *                      body _multistart_ray_roots surfaces.py:634-701)
 *   gwn_eval_rays      SPEC.md:381-407 winding_numbers_along_ray / slice /
 *                      voxelize: one intersection pass per ray, reused by
 *                      every point on it (ray reuse)
 *   gwn_solid_angle_many, gwn_ray_tris_hits
 *                      the mesh kernels of the dispatch layer
 *                      (_kernels.py:366, :443, :466): mesh solid angles and
 *                      ray/mesh all-hits
 *   gwn_single_loop_batch
 *                      _kernels.single_loop_batch (_kernels.py:801-823): the
 *                      kernel dispatch layer's ray-reuse boundary kernel
 *   gwn_last_error     error text; negative return codes map to the
 *                      GwnError hierarchy (errors.py:9-90) in the wrapper
 *
 * Threading: a scene is immutable after creation.  gwn_eval
 * may run concurrently from distinct host threads (its workspace is a
 * per-host-thread, per-device cache grown on demand, and each call
 * synchronises its stream before returning).  gwn_last_error is
 * thread-local.
 */
#ifndef GWN_B200_H
#define GWN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GWN_ABI_VERSION 6

/* return codes (negative = error) */
#define GWN_OK 0
#define GWN_E_INVALID -1      /* bad argument            -> ValueError / SceneError */
#define GWN_E_CUDA -2         /* CUDA runtime failure    -> GwnError */
#define GWN_E_NODEVICE -3     /* no usable sm_100 device -> GwnError */
#define GWN_E_OOM -4          /* device allocation       -> GwnError */

/* per-query status (int8) written by gwn_eval */
#define GWN_STATUS_OK 0
#define GWN_STATUS_ON_SURFACE 1   /* OnSurface: jittered by jitter_scale*diag */
#define GWN_STATUS_EXHAUSTED 2    /* SeedExhausted: re-shoot budget spent     */
#define GWN_STATUS_DEGENERATE 3   /* DegenerateProjection: jittered           */
#define GWN_STATUS_JITTER_EXHAUSTED 4 /* still on the surface / boundary after
                                     max_jitters jitters: w is unreliable   */

/* gwn_eval flags */
#define GWN_HOST_BUFFERS 1        /* queries / outputs are host pointers */

/* Mirrors reference EpsilonConfig (config.py:15-38) + engine knobs. */
typedef struct gwn_params {
  double residual;          /* config.py:29  accepted |f(u,v)-O-tD|      1e-10 */
  double dedup;             /* config.py:28  root merge distance         1e-9  */
  double tangent;           /* config.py:25  tangent_parametric          1e-12 */
  double edge_graze;        /* config.py:27  grazing distance            1e-10 */
  double degenerate;        /* config.py:18  projection degeneracy       1e-12 */
  double jitter_scale;      /* config.py:33  jitter, x scene diagonal    1e-7  */
  double domain_tol;        /* surfaces.py:668 domain_contains tolerance 1e-9  */
  double t_tol;             /* surfaces.py:670 t >= -t_tol               1e-12 */
  double on_surface_t;      /* |t| of a hit that means "on the surface" 1e-9  */
  double band_factor;       /* polyline/curve band safety factor         2.0   */
  int32_t samples_per_edge; /* surfaces.py:611 boundary samples          200   */
  int32_t max_rounds;       /* SPEC.md:320 ray re-shoot budget           32    */
  int32_t max_jitters;      /* SPEC.md:375 jitter budget                 3     */
  int32_t chunk_queries;    /* queries per internal chunk (0 = auto)           */
  uint64_t dir_seed;        /* deterministic direction sequence seed           */
  int32_t cached_rounds;    /* direction rounds kept on the scene (>= 1; later
                               re-shoot rounds are built per eval and freed) 4 */
  int32_t reserved_;
} gwn_params;

typedef struct gwn_scene gwn_scene;

typedef struct gwn_scene_info {
  int64_t n_patches;
  int64_t n_net_edges;      /* boundary edge curves left after cancellation */
  int64_t n_net_segments;   /* polyline segments the boundary term sums     */
  double bbox_min[3];
  double bbox_max[3];
  double diag;
  int32_t device;
  int32_t sm_count;
  int64_t n_far_cycles;     /* boundary cycles with a far-field expansion    */
  int32_t fmm_levels;       /* leaf level of round 0's local-expansion octree
                               (0: per-pair far field only)                  */
  int32_t pad_;
  int64_t fmm_translations; /* (box, cycle) multipole-to-local translations  */
  int64_t fmm_leftover;     /* entries left to the per-query path, all leaves */
  double fmm_build_ms;      /* host wall time of the octree build (scene creation) */
} gwn_scene_info;

/* Device-side counters of the last gwn_eval on a scene (for the roofline
 * and the divergence analysis). */
typedef struct gwn_stats {
  int64_t queries;
  int64_t rounds;           /* direction rounds run (all chunks)           */
  int64_t retried;          /* query re-evaluations beyond round 0         */
  int64_t candidates;       /* (query, patch) pairs surviving the cull     */
  int64_t nodes;            /* subdivision nodes tested in the intersector */
  int64_t newton_iters;
  int64_t roots;
  int64_t boundary_segments;/* (query, net segment) pairs evaluated        */
  int64_t kernel_launches;
  double ms_cull, ms_intersect, ms_boundary, ms_other;  /* event timings, 0 if not timed */
  double ms_k3_candidates, ms_k3_fallback, ms_k3_newton;  /* split of ms_intersect;
                                 candidates: the candidate test plus, for scenes past the
                                 shared-memory patch table, the patch-bin scan and scatter
                                 that order the Newton queue; newton: the Newton kernel */
  int64_t k3_fallback_items;  /* undecided leaf candidates solved by the DFS fallback */
  int64_t k3_newton_items;    /* certified leaf candidates (Newton solves)          */
  int64_t far_pairs;          /* (query, boundary cycle) pairs taken by the far-field
                                 expansion instead of the exact fan sum */
  int64_t far_terms;          /* solid-harmonic terms those expansions summed          */
  int64_t near_pairs;         /* (query, boundary cycle) pairs summed exactly          */
  double ms_k4_far, ms_k4_exact;  /* split of ms_boundary (far-field scenes, timed)   */
  int64_t rounds_built;       /* direction rounds (K1 structures) cached on the scene */
  double ms_round_build;      /* host wall time building new rounds in this eval      */
  int64_t local_evals;        /* queries whose far field came from a leaf's local expansion */
  int64_t shadow_pairs;       /* far pairs whose forward half-line crosses the cycle's
                                 sphere (expansion + shadow winding number, DESIGN §9 f4) */
} gwn_stats;

int gwn_abi_version(void);
const char* gwn_last_error(void);
void gwn_params_default(gwn_params* p);

/* Copy n_patches bicubic control nets ((P,4,4,3) f64, i = u index) to
 * `device`, build the net boundary and the round-0 patch hierarchy. */
int gwn_scene_create(const double* ctrl, int64_t n_patches, const gwn_params* prm,
                     int device, gwn_scene** out);
int gwn_scene_destroy(gwn_scene* scene);
int gwn_scene_info_get(const gwn_scene* scene, gwn_scene_info* out);

/* w[i] = generalized winding number of queries[i] ((n,3) f64), status[i] as
 * above.  `index_base` is the global id of queries[0] (jitter hash; keeps
 * sharded results identical to unsharded).  stream = cudaStream_t or NULL. */
int gwn_eval(gwn_scene* scene, const double* queries, int64_t n, int64_t index_base,
             double* w_out, int8_t* status_out, int32_t flags, void* stream);

/* Stats of the last gwn_eval on this scene; `timed` != 0 on the next eval
 * records per-kernel CUDA-event times (adds event syncs). */
int gwn_stats_get(const gwn_scene* scene, gwn_stats* out);

/* Ray reuse (SPEC.md:381-407 winding_numbers_along_ray / slice / voxelize;
 * PAPER.md:305-307): R parallel rays o_r + t d, sharing `direction`; ray r
 * carries the sorted parameters ts[offs[r] .. offs[r+1]) (offs has R+1
 * entries, offs[0] = 0).  One intersection pass per RAY; each point takes
 * chi from the cached hits beyond it plus its own boundary term.  Points on
 * rays with a tangent / grazing hit, clashing with a hit, degenerate or in
 * the band are re-evaluated by the per-point engine (same status codes as
 * gwn_eval; jitter keyed by the point's global index).  *rays_cast (may be
 * NULL) receives the number of intersection rays cast (= R). */
int gwn_eval_rays(gwn_scene* scene, const double* origins, int64_t R,
                  const double direction[3], const double* ts, const int64_t* offs,
                  double* w_out, int8_t* status_out, int32_t flags, void* stream,
                  int64_t* rays_cast);
int gwn_set_timing(gwn_scene* scene, int32_t timed);

/* patch.all_hits(ray, t_window, eps) (surfaces.py:587-589, body
 * surfaces.py:634-701): all hits of one ray with one patch of the scene, host
 * buffers.  `eps` = the caller's thresholds (NULL: the scene's); only roots
 * with t in [t_lo, t_hi] (+-1e-12, surfaces.py:679) are returned, sorted by t.
 * Records: t, u, v, sign, tangency, grazing.  A near-tangent contact the
 * subdivision cannot separate is returned as a tangent record.  Returns the
 * count (at most 18, Bezout's bound for a line and a bicubic; only `cap`
 * rows written) or a negative error; *flags_out (may be NULL) receives the
 * root set's flag bits (1 = re-shoot: tangent / grazing contact). */
int gwn_all_hits(gwn_scene* scene, int64_t patch, const double origin[3],
                 const double direction[3], const gwn_params* eps, double t_lo,
                 double t_hi, double* t_out, double* uv_out, int32_t* sign_out,
                 int8_t* tangency_out, int8_t* grazing_out, int32_t cap,
                 int32_t* flags_out);

/* _kernels.single_loop_batch on the GPU: closed loop (B,3), ray, cached hit
 * ts/signs (H), query ts (K) -> w (K), ok (K).  Host buffers. */
int gwn_single_loop_batch(const double* loop_pts, int64_t B, const double origin[3],
                          const double direction[3], const double* hit_ts,
                          const int64_t* hit_signs, int64_t H, const double* query_ts,
                          int64_t K, double on_tol, double t_eps, double* w_out,
                          int8_t* ok_out, int device);

/* ---- the rest of the kernel dispatch layer (pkg/src/gwn/_kernels.py) ----
 * Host buffers in and out; numpy-twin semantics (the numba kernels share the
 * broken _cross helper, _kernels.py:45). */

/* solid_angle_many / solid_angle_sum (_kernels.py:443-475): for each point
 * P[k] the signed solid angle sum_f 2 atan2(num, den) of the triangles
 * (V (nV,3) f64, T (nT,3) int64) -- NOT divided by 4 pi -- and
 * on_surface[k] = 1 when P[k] is on (or numerically on) the surface; those
 * triangles are left out of the sum (:405-411). */
int gwn_solid_angle_many(const double* V, int64_t nV, const int64_t* T, int64_t nT,
                         const double* P, int64_t nP, double guard, double* out,
                         int8_t* on_surface, int device);

/* The reference's Bvh (surfaces.py:74-163, build_bvh): node arrays and the
 * per-triangle Moller-Trumbore data, all host pointers, C-contiguous. */
typedef struct gwn_tri_bvh {
  const double* node_min;     /* (N,3) */
  const double* node_max;     /* (N,3) */
  const int64_t* node_left;   /* (N) -1 for leaves */
  const int64_t* node_right;  /* (N) */
  const int64_t* node_start;  /* (N) */
  const int64_t* node_count;  /* (N) */
  const int64_t* tri_order;   /* (F) */
  int64_t n_nodes;
  const double* V0;           /* (F,3) */
  const double* E1;           /* (F,3) */
  const double* E2;           /* (F,3) */
  const double* NN;           /* (F) |e1 x e2| */
  const double* NH;           /* (F,3) unit normals */
  const double* C;            /* (F,3) centroids */
  const double* R2;           /* (F) squared circumradii about the centroid */
  int64_t n_tris;
} gwn_tri_bvh;

/* bvh_ray_all_hits (_kernels.py:366-381) for R rays at once: hits of ray r
 * are [offs[r], offs[r+1]) (offs has R+1 entries, always written), in the
 * numpy twin's order (regular hits by triangle, then parallel contacts by
 * triangle; _kernels.py:312-363).  Returns the total hit count; the hit
 * arrays are written only when total <= cap (call again with cap = total
 * otherwise).  Negative on error. */
int64_t gwn_ray_tris_hits(const gwn_tri_bvh* bvh, const double* origins, const double* dirs,
                          int64_t R, double t_lo, double t_hi, double tang_eps,
                          double plane_tol, int64_t* offs, double* ts, int64_t* tris,
                          double* dotdn, double* us, double* vs, int64_t cap, int device);

/* Free this host thread's cached eval workspace on `device` (gwn_eval keeps
 * its buffers at the largest batch seen, for the next call). */
int gwn_release_caches(int device);

/* Host-side helpers shared with the oracle contract (no device needed). */
void gwn_direction(uint64_t seed, int32_t round, double d[3]);
void gwn_jitter_dir(uint64_t seed, int64_t qidx, int32_t attempt, double v[3]);
int64_t gwn_net_boundary(const double* ctrl, int64_t n_patches, double* out_ctrl,
                         int32_t* out_weight);

/* FP64 peak microbenchmark (DFMA chains on every SM), TFLOP/s. */
int gwn_fp64_peak(int device, double* tflops, double* ms);

/* Max ulp error of K4's reciprocal square root over a log-uniform sweep. */
int gwn_selftest_rsqrt(int device, int64_t n, uint64_t* max_ulp);

#ifdef __cplusplus
}
#endif
#endif
