/* oracle/gwn_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's winding-number path for bicubic Bezier
 * patches (arXiv 2408.04466 reference, /root/reference/pkg/src/gwn).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load libgwn_oracle.so, and only as the checker or the
 * timed CPU baseline -- never as the product path.
 *
 * Pinning: tests/golden/ fixtures are produced by tests/golden/make_golden.py,
 * which imports the reference itself (gwn.geometry.ray_aabb_clip,
 * gwn.surfaces._multistart_ray_roots / patch_boundary through a bicubic
 * adapter of the reference patch protocol, gwn._kernels.single_loop_batch
 * from a scratch copy with the one-line _cross fix at _kernels.py:45, and the
 * numpy solid-angle twin _kernels.py:422-440 for tessellation adjudication).
 * tests/test_oracle_golden.py checks this library against every fixture.
 */
#ifndef GWN_ORACLE_H
#define GWN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors reference EpsilonConfig (pkg/src/gwn/config.py:15-38) plus the
 * engine knobs of SPEC.md:371-380,427 and the boundary sampling of
 * surfaces.py:611 (samples_per_edge). */
typedef struct or_params {
  double residual;        /* config.py:29  1e-10 */
  double dedup;           /* config.py:28  1e-9  */
  double tangent;         /* config.py:25  1e-12 (tangent_parametric) */
  double edge_graze;      /* config.py:27  1e-10 */
  double degenerate;      /* config.py:18  1e-12 */
  double jitter_scale;    /* config.py:33  1e-7  */
  double domain_tol;      /* surfaces.py:668  1e-9 */
  double t_tol;           /* surfaces.py:670  1e-12 */
  double on_surface_t;    /* |t| of a hit below which the query is on the surface */
  double band_factor;     /* safety factor of the polyline/curve band test */
  int32_t samples_per_edge; /* surfaces.py:472,584,611  200 */
  int32_t max_rounds;       /* SPEC.md:320 retry budget 32 */
  int32_t max_jitters;      /* SPEC.md:373-375 jitter budget 3 */
  int32_t subdiv_depth;     /* de Casteljau levels before the multistart solve */
  uint64_t dir_seed;
} or_params;

typedef struct or_record {  /* surfaces.py:33-48 IntersectionRecord */
  double t, u, v;
  double normal[3];
  int32_t sign, tangency, grazing, pad;
} or_record;

void or_params_default(or_params* p);

/* geometry.py:198-219 ray_aabb_clip; returns 1 and the window, 0 on miss. */
int or_ray_aabb_clip(const double o[3], const double d[3], const double bmin[3],
                     const double bmax[3], double* t0, double* t1);

/* bicubic point / partials, ctrl (4,4,3) row-major, i = u index. */
void or_bicubic_point(const double* ctrl, double u, double v, double out[3]);
void or_bicubic_partials(const double* ctrl, double u, double v, double fu[3], double fv[3]);

/* surfaces.py:634-701 on the whole patch domain with the reference seeding
 * (domain-centre seeds), Newton standing in for MINPACK hybr.  Returns the
 * number of records written (<= cap), sorted by t. */
int or_multistart_hits(const double* ctrl, const double o[3], const double d[3],
                       const or_params* prm, or_record* out, int cap);

/* Same acceptance rules, seeds from `depth` levels of de Casteljau
 * sub-patches whose control boxes the ray clips. */
int or_patch_all_hits(const double* ctrl, const double o[3], const double d[3],
                      const or_params* prm, or_record* out, int cap);

/* surfaces.py:611-626 patch_boundary: 4(S-1) points, CCW in the domain. */
void or_patch_boundary(const double* ctrl, int S, double* out_pts);

/* Fan-formula boundary term of one closed loop seen from p
 * with ray direction d; equals single_loop_batch's w - chi where ok=1. */
double or_loop_fan(const double* loop_pts, int64_t n, const double p[3], const double d[3]);

/* Net boundary: shared edge curves cancelled exactly.  Returns the number of
 * net edges; if out_ctrl != NULL writes (n,4,3) control points in effective
 * direction and out_weight (n) multiplicities. */
int64_t or_net_boundary(const double* ctrl, int64_t n_patches, double* out_ctrl,
                        int32_t* out_weight);

/* Cubic edge sampling used by both the oracle and the GPU net boundary. */
void or_sample_edge(const double* ctrl4, int S, double* out);

/* Deterministic ray direction for round r and the jitter offset direction. */
void or_direction(uint64_t seed, int32_t round, double d[3]);
void or_jitter_dir(uint64_t seed, int64_t qidx, int32_t attempt, double v[3]);

/* Whole engine: per query w and status
 * (0 ok, 1 on-surface after jitter, 2 retries exhausted, 3 degenerate
 * projection after jitter).  qidx (nullable) gives global query ids for the
 * jitter hash.  chi_out / rounds_out nullable.  Threads: nthreads<=0 -> all. */
int or_scene_eval(const double* ctrl, int64_t n_patches, const double* queries,
                  const int64_t* qidx, int64_t n, const or_params* prm,
                  double* w_out, int8_t* status_out, int32_t* chi_out,
                  int32_t* rounds_out, int nthreads);

/* One round at a fixed direction without retries: chi, boundary term,
 * flag bits (1 tangent/grazing, 2 band, 4 on-surface, 8 degenerate). */
int or_scene_eval_dir(const double* ctrl, int64_t n_patches, const double* queries,
                      int64_t n, const double d[3], const or_params* prm,
                      int32_t* chi_out, double* bterm_out, int32_t* flags_out,
                      int nthreads);

#ifdef __cplusplus
}
#endif
#endif
