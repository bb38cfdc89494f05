/* oracle/gwn_oracle.c -- TEST INFRASTRUCTURE ONLY (see gwn_oracle.h).
 *
 * CPU restatement of the reference path, used as the parity checker for the
 * CUDA product and as the timed CPU baseline.  Every function cites the
 * reference file:line it follows (paths relative to
 * /root/reference/pkg/src/gwn/ unless noted).  Compiled with
 * -ffp-contract=off so edge sampling is bit-identical to the product's
 * explicitly-rounded device sampler.
 *
 * Third-party arithmetic: the reference solves f(u,v) - O - tD = 0 with
 * scipy.optimize.root(method="hybr") (MINPACK hybrj; scipy>=1.10 per
 * pkg/pyproject.toml:12, 1.18.1 installed where the fixtures were made),
 * called at surfaces.py:661.  We restate it as damped Newton with the same
 * xtol (1e-14) and the reference's own acceptance tests (surfaces.py:664-675);
 * root sets are pinned against the reference's outputs by the golden tests.
 */
#include "gwn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define OR_PI 3.14159265358979323846
#define OR_MAX_ROOTS 64

/* ------------------------------------------------------------------------- */
/* parameters                                                                */
/* ------------------------------------------------------------------------- */

void or_params_default(or_params* p) {
  p->residual = 1e-10;     /* config.py:29 */
  p->dedup = 1e-9;         /* config.py:28 */
  p->tangent = 1e-12;      /* config.py:25 */
  p->edge_graze = 1e-10;   /* config.py:27 */
  p->degenerate = 1e-12;   /* config.py:18 */
  p->jitter_scale = 1e-7;  /* config.py:33 */
  p->domain_tol = 1e-9;    /* surfaces.py:668 */
  p->t_tol = 1e-12;        /* surfaces.py:670 */
  p->on_surface_t = 1e-9;  /* SPEC.md:383 "within 1e-9 (else perturbed)" */
  p->band_factor = 2.0;
  p->samples_per_edge = 200; /* surfaces.py:611 */
  p->max_rounds = 32;
  p->max_jitters = 3;
  p->subdiv_depth = 3;       /* 8x8 sub-patches recover all roots */
  p->dir_seed = 0x2408044660ull;
}

/* ------------------------------------------------------------------------- */
/* small vector helpers                                                      */
/* ------------------------------------------------------------------------- */

static inline double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
static inline void cross3(const double* a, const double* b, double* c) {
  /* the correct z component; the reference numba helper has ay*bz here
   * (_kernels.py:45), which is the documented bug we do NOT restate */
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
static inline double norm3(const double* a) { return sqrt(dot3(a, a)); }

/* ------------------------------------------------------------------------- */
/* deterministic sequences (shared contract with the product)     */
/* ------------------------------------------------------------------------- */

static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

void or_direction(uint64_t seed, int32_t round, double d[3]) {
  uint64_t s = seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(round + 1));
  double z = 1.0 - 2.0 * u01(splitmix64(&s));
  double phi = 2.0 * OR_PI * u01(splitmix64(&s));
  double r = sqrt(fmax(0.0, 1.0 - z * z));
  d[0] = r * cos(phi);
  d[1] = r * sin(phi);
  d[2] = z;
}

void or_jitter_dir(uint64_t seed, int64_t qidx, int32_t attempt, double v[3]) {
  uint64_t s = seed ^ 0x5851F42D4C957F2Dull;
  s ^= (uint64_t)qidx * 0x9E3779B97F4A7C15ull;
  s ^= (uint64_t)(attempt + 1) * 0xC2B2AE3D27D4EB4Full;
  double x = 2.0 * u01(splitmix64(&s)) - 1.0;
  double y = 2.0 * u01(splitmix64(&s)) - 1.0;
  double z = 2.0 * u01(splitmix64(&s)) - 1.0;
  double n = sqrt(x * x + y * y + z * z);
  if (n < 1e-3) { v[0] = 1.0; v[1] = 0.0; v[2] = 0.0; return; }
  v[0] = x / n; v[1] = y / n; v[2] = z / n;
}

/* ------------------------------------------------------------------------- */
/* geometry.py:198-219 ray_aabb_clip                                          */
/* ------------------------------------------------------------------------- */

int or_ray_aabb_clip(const double o[3], const double d[3], const double lo[3],
                     const double hi[3], double* tmin_out, double* tmax_out) {
  double t_min = 0.0, t_max = INFINITY;          /* geometry.py:203 */
  for (int k = 0; k < 3; ++k) {                   /* geometry.py:204 */
    if (d[k] == 0.0) {                            /* geometry.py:207-210 */
      if (o[k] < lo[k] || o[k] > hi[k]) return 0;
      continue;
    }
    double inv = 1.0 / d[k];                      /* geometry.py:211 */
    double t0 = (lo[k] - o[k]) * inv, t1 = (hi[k] - o[k]) * inv;
    if (t0 > t1) { double tt = t0; t0 = t1; t1 = tt; }
    t_min = fmax(t_min, t0);                      /* geometry.py:215-216 */
    t_max = fmin(t_max, t1);
    if (t_max < t_min) return 0;                  /* geometry.py:217-218 */
  }
  *tmin_out = t_min;
  *tmax_out = t_max;
  return 1;
}

/* ------------------------------------------------------------------------- */
/* bicubic adapter of the patch protocol (template: CoonsPatch,              */
/* surfaces.py:499-589)                                                      */
/* ------------------------------------------------------------------------- */

static inline void bern(double t, double b[4]) {
  double s = 1.0 - t;
  b[0] = s * s * s; b[1] = 3.0 * t * s * s; b[2] = 3.0 * t * t * s; b[3] = t * t * t;
}
static inline void dbern(double t, double b[4]) {
  double s = 1.0 - t;
  b[0] = -3.0 * s * s; b[1] = 3.0 * s * s - 6.0 * t * s;
  b[2] = 6.0 * t * s - 3.0 * t * t; b[3] = 3.0 * t * t;
}

void or_bicubic_point(const double* X, double u, double v, double out[3]) {
  double bu[4], bv[4];
  bern(u, bu); bern(v, bv);
  out[0] = out[1] = out[2] = 0.0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double w = bu[i] * bv[j];
      const double* x = X + (i * 4 + j) * 3;
      out[0] += w * x[0]; out[1] += w * x[1]; out[2] += w * x[2];
    }
}

void or_bicubic_partials(const double* X, double u, double v, double fu[3], double fv[3]) {
  double bu[4], bv[4], du[4], dv[4];
  bern(u, bu); bern(v, bv); dbern(u, du); dbern(v, dv);
  fu[0] = fu[1] = fu[2] = fv[0] = fv[1] = fv[2] = 0.0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const double* x = X + (i * 4 + j) * 3;
      double a = du[i] * bv[j], b = bu[i] * dv[j];
      for (int k = 0; k < 3; ++k) { fu[k] += a * x[k]; fv[k] += b * x[k]; }
    }
}

static void aabb_of(const double* pts, int n, double lo[3], double hi[3]) {
  /* geometry.py:70-73 Aabb.of_points */
  for (int k = 0; k < 3; ++k) { lo[k] = pts[k]; hi[k] = pts[k]; }
  for (int i = 1; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], pts[3 * i + k]);
      hi[k] = fmax(hi[k], pts[3 * i + k]);
    }
}

static inline double domain_boundary_dist(double u, double v) {
  /* surfaces.py:578-579 */
  return fmin(fmin(u, 1.0 - u), fmin(v, 1.0 - v));
}

/* ------------------------------------------------------------------------- */
/* the solver: stand-in for scipy root(hybr) at surfaces.py:651-663          */
/* ------------------------------------------------------------------------- */

static void fun3(const double* X, const double o[3], const double d[3], const double x[3],
                 double F[3]) {
  double p[3];
  or_bicubic_point(X, x[0], x[1], p);             /* surfaces.py:651-652 */
  for (int k = 0; k < 3; ++k) F[k] = p[k] - o[k] - x[2] * d[k];
}

static int solve3(const double J[3][3], const double b[3], double x[3]) {
  /* Gaussian elimination with partial pivoting */
  double A[3][4];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) A[r][c] = J[r][c];
    A[r][3] = b[r];
  }
  for (int c = 0; c < 3; ++c) {
    int piv = c;
    for (int r = c + 1; r < 3; ++r)
      if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
    if (A[piv][c] == 0.0) return 0;
    if (piv != c)
      for (int k = 0; k < 4; ++k) { double t = A[c][k]; A[c][k] = A[piv][k]; A[piv][k] = t; }
    for (int r = c + 1; r < 3; ++r) {
      double f = A[r][c] / A[c][c];
      for (int k = c; k < 4; ++k) A[r][k] -= f * A[c][k];
    }
  }
  for (int r = 2; r >= 0; --r) {
    double s = A[r][3];
    for (int k = r + 1; k < 3; ++k) s -= A[r][k] * x[k];
    x[r] = s / A[r][r];
  }
  return isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
}

static void newton3(const double* X, const double o[3], const double d[3], double x[3]) {
  double F[3];
  fun3(X, o, d, x, F);
  double nf = norm3(F);
  for (int it = 0; it < 100; ++it) {
    double fu[3], fv[3], J[3][3], rhs[3], step[3];
    or_bicubic_partials(X, x[0], x[1], fu, fv);   /* surfaces.py:654-656 */
    for (int k = 0; k < 3; ++k) {
      J[k][0] = fu[k]; J[k][1] = fv[k]; J[k][2] = -d[k];
      rhs[k] = -F[k];
    }
    if (!solve3(J, rhs, step)) return;
    double lam = 1.0, xn[3], Fn[3], nfn = 0.0;
    int accepted = 0;
    for (int ls = 0; ls < 12; ++ls) {
      for (int k = 0; k < 3; ++k) xn[k] = x[k] + lam * step[k];
      fun3(X, o, d, xn, Fn);
      nfn = norm3(Fn);
      if (nfn < nf || nfn == 0.0) { accepted = 1; break; }
      lam *= 0.5;
    }
    if (!accepted) return;
    double dx = lam * norm3(step), xs = norm3(x);
    for (int k = 0; k < 3; ++k) { x[k] = xn[k]; F[k] = Fn[k]; }
    nf = nfn;
    if (dx <= 1e-14 * (xs + 1e-14)) return;        /* xtol=1e-14, surfaces.py:662 */
  }
}

/* ------------------------------------------------------------------------- */
/* surfaces.py:634-701 _multistart_ray_roots (root collection + records)     */
/* ------------------------------------------------------------------------- */

typedef struct roots_t {
  int n;
  int ambiguous;      /* a leaf at the depth cap stayed uncertified (a fold) */
  double amb_t;
  double r[OR_MAX_ROOTS][3];
} roots_t;

static void try_seed(const double* X, const double o[3], const double d[3], const or_params* prm,
                     double u0, double v0, double t_seed, roots_t* R) {
  double x[3] = {u0, v0, t_seed};                  /* surfaces.py:660-661 */
  newton3(X, o, d, x);
  double F[3];
  fun3(X, o, d, x, F);                             /* surfaces.py:664 */
  if (!(norm3(F) <= prm->residual)) return;        /* surfaces.py:665-666 */
  double u = x[0], v = x[1], t = x[2];
  double tol = prm->domain_tol;                    /* surfaces.py:668 domain_contains */
  if (!(u >= -tol && u <= 1.0 + tol && v >= -tol && v <= 1.0 + tol)) return;
  if (t < -prm->t_tol) return;                     /* surfaces.py:670 */
  double pt[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
  for (int i = 0; i < R->n; ++i) {                 /* surfaces.py:672-674 */
    double q[3], diff[3];
    for (int k = 0; k < 3; ++k) { q[k] = o[k] + R->r[i][2] * d[k]; diff[k] = pt[k] - q[k]; }
    if (norm3(diff) < prm->dedup) return;
  }
  if (R->n < OR_MAX_ROOTS) {
    R->r[R->n][0] = u; R->r[R->n][1] = v; R->r[R->n][2] = t;
    R->n++;
  }
}

static void multistart_box(const double* X, const double o[3], const double d[3],
                           const or_params* prm, const double lo[3], const double hi[3],
                           double uc, double vc, roots_t* R) {
  double c0, c1;
  if (!or_ray_aabb_clip(o, d, lo, hi, &c0, &c1)) return;   /* surfaces.py:636-639 */
  double t_lo = fmax(c0, 0.0), t_hi = c1;                   /* surfaces.py:640-643 */
  if (t_hi < t_lo) return;
  double diag[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  double dg = fmax(norm3(diag), 1e-12);                     /* surfaces.py:644 */
  double ns = ceil(30.0 * (t_hi - t_lo) / dg);              /* surfaces.py:645 */
  int n_seeds = ns < 2.0 ? 2 : (ns > 4096.0 ? 4096 : (int)ns);
  for (int k = 0; k < n_seeds; ++k) {                       /* surfaces.py:659-660 */
    double t_seed = t_lo + (k + 0.5) * (t_hi - t_lo) / n_seeds;
    try_seed(X, o, d, prm, uc, vc, t_seed, R);
  }
}

static int build_records(const double* X, const double d[3],
                         const or_params* prm, const roots_t* R, or_record* out, int cap) {
  int n = 0;
  for (int i = 0; i < R->n && n < cap; ++i) {      /* surfaces.py:678 */
    double u = R->r[i][0], v = R->r[i][1], t = R->r[i][2];
    if (t < 0.0 - 1e-12) continue;                 /* surfaces.py:679-680 */
    double fu[3], fv[3], nn[3];
    or_bicubic_partials(X, u, v, fu, fv);          /* surfaces.py:681 */
    cross3(fu, fv, nn);                            /* surfaces.py:682 */
    double len = norm3(nn);
    or_record* rec = &out[n++];
    rec->t = t; rec->u = u; rec->v = v; rec->pad = 0;
    if (len < prm->degenerate) {                   /* surfaces.py:684-687 */
      rec->normal[0] = d[0]; rec->normal[1] = d[1]; rec->normal[2] = d[2];
      rec->sign = 1; rec->tangency = 1; rec->grazing = 1;
      continue;
    }
    for (int k = 0; k < 3; ++k) rec->normal[k] = nn[k] / len;   /* surfaces.py:688 */
    double dd = dot3(d, rec->normal);                           /* surfaces.py:689 */
    rec->sign = dd > 0.0 ? 1 : -1;                              /* surfaces.py:695 */
    rec->tangency = fabs(dd) <= prm->tangent;                   /* surfaces.py:696 */
    rec->grazing = domain_boundary_dist(u, v) < prm->edge_graze; /* surfaces.py:697 */
  }
  /* surfaces.py:700 sort by t (insertion sort, tiny n) */
  for (int i = 1; i < n; ++i) {
    or_record key = out[i];
    int j = i - 1;
    while (j >= 0 && out[j].t > key.t) { out[j + 1] = out[j]; --j; }
    out[j + 1] = key;
  }
  return n;
}

int or_multistart_hits(const double* X, const double o[3], const double d[3],
                       const or_params* prm, or_record* out, int cap) {
  double lo[3], hi[3];
  aabb_of(X, 16, lo, hi);                          /* surfaces.py:636 (control-net box) */
  roots_t R;
  R.n = 0;
  R.ambiguous = 0;
  R.amb_t = 0.0;
  multistart_box(X, o, d, prm, lo, hi, 0.5, 0.5, &R);   /* domain_center, surfaces.py:581 */
  return build_records(X, d, prm, &R, out, cap);
}

/* de Casteljau halving of a 4x4 net along u (dir=0) or v (dir=1) */
static void split_net(const double* N, int dir, double* A, double* B) {
  for (int l = 0; l < 4; ++l) {
    double p[4][3];
    for (int m = 0; m < 4; ++m) {
      const double* src = dir == 0 ? N + (m * 4 + l) * 3 : N + (l * 4 + m) * 3;
      for (int k = 0; k < 3; ++k) p[m][k] = src[k];
    }
    double q[7][3];
    for (int k = 0; k < 3; ++k) {
      double a01 = 0.5 * (p[0][k] + p[1][k]), a12 = 0.5 * (p[1][k] + p[2][k]);
      double a23 = 0.5 * (p[2][k] + p[3][k]);
      double b0 = 0.5 * (a01 + a12), b1 = 0.5 * (a12 + a23), c = 0.5 * (b0 + b1);
      q[0][k] = p[0][k]; q[1][k] = a01; q[2][k] = b0; q[3][k] = c;
      q[4][k] = b1; q[5][k] = a23; q[6][k] = p[3][k];
    }
    for (int m = 0; m < 4; ++m) {
      double* da = dir == 0 ? A + (m * 4 + l) * 3 : A + (l * 4 + m) * 3;
      double* db = dir == 0 ? B + (m * 4 + l) * 3 : B + (l * 4 + m) * 3;
      for (int k = 0; k < 3; ++k) { da[k] = q[m][k]; db[k] = q[m + 3][k]; }
    }
  }
}

/* Injectivity certificate for the ray projection of a sub-patch: the
 * projected f_u and f_v control vectors (onto the plane normal to d) must lie
 * in pointed cones whose lines (mod pi) are disjoint.  Then the averaged
 * Jacobian between any two points of the convex leaf is non-singular, so the
 * ray meets the leaf at most once and one Newton solve decides it. */
static int cone_of(const double* V, int n, const double e1[3], const double e2[3],
                   double* lo, double* hi) {
  double mx = 0.0, my = 0.0, x[12], y[12];
  for (int k = 0; k < n; ++k) {
    x[k] = dot3(V + 3 * k, e1);
    y[k] = dot3(V + 3 * k, e2);
    double l = sqrt(x[k] * x[k] + y[k] * y[k]);
    if (!(l > 1e-300)) return 0;
    mx += x[k] / l;
    my += y[k] / l;
  }
  double ml = sqrt(mx * mx + my * my);
  if (!(ml > 1e-12)) return 0;
  double c = atan2(my, mx), a = 0.0, b = 0.0;
  for (int k = 0; k < n; ++k) {
    double phi = atan2(mx * y[k] - my * x[k], mx * x[k] + my * y[k]);
    if (k == 0 || phi < a) a = phi;
    if (k == 0 || phi > b) b = phi;
  }
  if (a < -1.3 || b > 1.3) return 0;
  *lo = c + a;
  *hi = c + b;
  return 1;
}

static int leaf_injective(const double* N, const double d[3]) {
  double e1[3], e2[3], ax[3] = {0, 0, 0};
  int m = fabs(d[0]) < fabs(d[1]) ? (fabs(d[0]) < fabs(d[2]) ? 0 : 2) : (fabs(d[1]) < fabs(d[2]) ? 1 : 2);
  ax[m] = 1.0;
  cross3(d, ax, e1);
  double l = norm3(e1);
  for (int k = 0; k < 3; ++k) e1[k] /= l;
  cross3(d, e1, e2);
  double U[36], V[36];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 3; ++k) {
        U[(i * 4 + j) * 3 + k] = N[((i + 1) * 4 + j) * 3 + k] - N[(i * 4 + j) * 3 + k];
        V[(j * 3 + i) * 3 + k] = N[(j * 4 + i + 1) * 3 + k] - N[(j * 4 + i) * 3 + k];
      }
  double lo1, hi1, lo2, hi2;
  if (!cone_of(U, 12, e1, e2, &lo1, &hi1) || !cone_of(V, 12, e1, e2, &lo2, &hi2)) return 0;
  const double margin = 1e-6;
  for (int s = -3; s <= 3; ++s) {
    double sh = s * OR_PI;
    if (lo1 - margin <= hi2 + sh && lo2 + sh <= hi1 + margin) return 0;
  }
  return 1;
}

#define OR_MIN_DEPTH 3
#define OR_MAX_DEPTH 14

static void subdiv_hits(const double* X, const double* N, double u0, double v0, double w,
                        int depth, const double o[3], const double d[3], const or_params* prm,
                        roots_t* R) {
  double lo[3], hi[3], c0, c1;
  aabb_of(N, 16, lo, hi);                          /* geometry.py:70-73 */
  if (!or_ray_aabb_clip(o, d, lo, hi, &c0, &c1)) return;   /* geometry.py:198-219 */
  if (c1 < fmax(c0, 0.0)) return;
  const int certified = depth >= prm->subdiv_depth && leaf_injective(N, d);
  int leaf = depth >= OR_MAX_DEPTH || certified;
  if (leaf) {
    const int n_before = R->n;
    /* the reference seeding (domain centre, t seeds; surfaces.py:645-660)
     * on the leaf, plus the leaf's four quarter points at mid-window */
    multistart_box(X, o, d, prm, lo, hi, u0 + 0.5 * w, v0 + 0.5 * w, R);
    double tm = 0.5 * (fmax(c0, 0.0) + c1);
    for (int q = 0; q < 4; ++q)
      try_seed(X, o, d, prm, u0 + (q & 1 ? 0.75 : 0.25) * w, v0 + (q & 2 ? 0.75 : 0.25) * w,
               tm, R);
    if (!certified && !R->ambiguous) {
      /* an uncertified leaf at the depth cap (a silhouette fold) whose seeds
       * converged to a near-tangent contact: residual-accepted points along
       * a tangent are not a reliable root set.  As on the GPU
       * (undecided nodes, gwn_wavefront.cu), the ray is reported tangent and
       * the query is re-shot. */
      for (int i = n_before; i < R->n; ++i) {
        double fu[3], fv[3], nn[3];
        or_bicubic_partials(X, R->r[i][0], R->r[i][1], fu, fv);
        cross3(fu, fv, nn);
        const double l = norm3(nn);
        if (!(l > 0.0) || fabs(dot3(nn, d)) < 1e-4 * l) {
          R->ambiguous = 1;
          R->amb_t = R->r[i][2];
          break;
        }
      }
    }
    return;
  }
  double A[48], B[48], AA[48], AB[48], BA[48], BB[48];
  split_net(N, 0, A, B);
  split_net(A, 1, AA, AB);
  split_net(B, 1, BA, BB);
  double h = 0.5 * w;
  subdiv_hits(X, AA, u0, v0, h, depth + 1, o, d, prm, R);
  subdiv_hits(X, AB, u0, v0 + h, h, depth + 1, o, d, prm, R);
  subdiv_hits(X, BA, u0 + h, v0, h, depth + 1, o, d, prm, R);
  subdiv_hits(X, BB, u0 + h, v0 + h, h, depth + 1, o, d, prm, R);
}

int or_patch_all_hits(const double* X, const double o[3], const double d[3],
                      const or_params* prm, or_record* out, int cap) {
  roots_t R;
  R.n = 0;
  R.ambiguous = 0;
  R.amb_t = 0.0;
  subdiv_hits(X, X, 0.0, 0.0, 1.0, 0, o, d, prm, &R);
  int n = build_records(X, d, prm, &R, out, cap);
  /* a root with |d . n^| < 1e-6 lies within ~1e-6 of a tangent contact:
   * residual acceptance (1e-10) then admits a run of points along the
   * tangent, each counted (measured: 44 "roots" at |d . n^| ~ 1e-8 on one
   * ray); re-shoot instead, as the GPU's certification does */
  for (int i = 0; i < n && !R.ambiguous; ++i)
    if (!out[i].tangency && fabs(dot3(out[i].normal, d)) < 1e-6) {
      R.ambiguous = 1;
      R.amb_t = out[i].t;
    }
  if (R.ambiguous) {
    /* one tangent record (sign 0: chi unchanged) carries the re-shoot */
    int k = n;
    if (k < cap) {
      ++n;
    } else {
      k = cap - 1;
    }
    or_record* rec = &out[k];
    rec->t = R.amb_t; rec->u = rec->v = 0.5; rec->pad = 0;
    rec->normal[0] = d[0]; rec->normal[1] = d[1]; rec->normal[2] = d[2];
    rec->sign = 0; rec->tangency = 1; rec->grazing = 0;
  }
  return n;
}

/* ------------------------------------------------------------------------- */
/* boundary sampling: surfaces.py:611-626                                    */
/* ------------------------------------------------------------------------- */

void or_patch_boundary(const double* X, int S, double* out) {
  double step = 1.0 / (double)(S - 1);             /* np.linspace(0,1,S) */
  int n = 0;
  for (int e = 0; e < 4; ++e) {                    /* surfaces.py:622, domain_edges :566-573 */
    for (int k = 0; k < S - 1; ++k) {              /* linspace(...)[:-1] */
      double t = (double)k * step, u, v;
      switch (e) {
        case 0: u = t; v = 0.0; break;
        case 1: u = 1.0; v = t; break;
        case 2: u = 1.0 - t; v = 1.0; break;
        default: u = 0.0; v = 1.0 - t; break;
      }
      or_bicubic_point(X, u, v, out + 3 * n);      /* surfaces.py:625 */
      ++n;
    }
  }
}

void or_sample_edge(const double* P, int S, double* out) {
  double step = 1.0 / (double)(S - 1);
  for (int k = 0; k < S; ++k) {
    double t = (k == S - 1) ? 1.0 : (double)k * step;
    double s = 1.0 - t;
    double b0 = (s * s) * s, b1 = ((3.0 * t) * s) * s;
    double b2 = ((3.0 * t) * t) * s, b3 = (t * t) * t;
    for (int c = 0; c < 3; ++c)
      out[3 * k + c] = ((b0 * P[c] + b1 * P[3 + c]) + b2 * P[6 + c]) + b3 * P[9 + c];
  }
}

/* ------------------------------------------------------------------------- */
/* boundary term: fan formula == _kernels.py:752-796 w-chi  */
/* ------------------------------------------------------------------------- */

static inline double fan_segment(const double* xa, const double* xb, const double p[3],
                                 const double c[3], double degenerate, double band_h,
                                 int* flags, double band_factor) {
  double a[3] = {xa[0] - p[0], xa[1] - p[1], xa[2] - p[2]};
  double b[3] = {xb[0] - p[0], xb[1] - p[1], xb[2] - p[2]};
  double la = norm3(a), lb = norm3(b);
  if (la < degenerate || lb < degenerate) {        /* _kernels.py:541-542 DegenerateProjection */
    *flags |= 8;
    return 0.0;
  }
  for (int k = 0; k < 3; ++k) { a[k] /= la; b[k] /= lb; }
  /* van Oosterom-Strackee for the unit triangle (c, a, b), c = -d, in the
   * exactly equivalent shifted form u = a - d, v = b - d:
   *   1 + a.b + b.c + c.a = u.v,   c.(a x b) = -d.(u x v)
   * which stays accurate when d points at the segment (u, v small). */
  double d[3] = {-c[0], -c[1], -c[2]};
  double u[3] = {a[0] - d[0], a[1] - d[1], a[2] - d[2]};
  double v[3] = {b[0] - d[0], b[1] - d[1], b[2] - d[2]};
  double uv[3];
  cross3(u, v, uv);
  double num = -dot3(d, uv);
  double den = dot3(u, v);
  if (den < 0.0 && band_h > 0.0) {
    double seg[3] = {xb[0] - xa[0], xb[1] - xa[1], xb[2] - xa[2]};
    double dist = fmin(la, lb) - norm3(seg);
    double ab[3];
    cross3(a, b, ab);
    double s2 = dot3(ab, ab);
    if (dist <= 0.0) {
      *flags |= 2;
    } else {
      double th = band_factor * band_h / dist;
      if (num * num <= th * th * s2) *flags |= 2;
    }
  }
  return 2.0 * atan2(num, den);
}

double or_loop_fan(const double* pts, int64_t n, const double p[3], const double d[3]) {
  double c[3] = {-d[0], -d[1], -d[2]};
  double total = 0.0;
  int flags = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = (i + 1 < n) ? i + 1 : 0;
    total += fan_segment(pts + 3 * i, pts + 3 * j, p, c, 1e-12, 0.0, &flags, 0.0);
  }
  return total / (4.0 * OR_PI);
}

/* ------------------------------------------------------------------------- */
/* net boundary (exact cancellation of shared edge curves)                   */
/* ------------------------------------------------------------------------- */

typedef struct edge_t {
  double c[12];
  int32_t w;
} edge_t;

static int cmp12(const double* a, const double* b) {
  for (int k = 0; k < 12; ++k) {
    if (a[k] < b[k]) return -1;
    if (a[k] > b[k]) return 1;
  }
  return 0;
}
static int cmp_edge(const void* x, const void* y) {
  return cmp12(((const edge_t*)x)->c, ((const edge_t*)y)->c);
}

static void patch_edge(const double* X, int e, double out[12]) {
  for (int m = 0; m < 4; ++m) {
    int i, j;
    switch (e) {
      case 0: i = m; j = 0; break;          /* (t, 0)   */
      case 1: i = 3; j = m; break;          /* (1, t)   */
      case 2: i = 3 - m; j = 3; break;      /* (1-t, 1) */
      default: i = 0; j = 3 - m; break;     /* (0, 1-t) */
    }
    for (int k = 0; k < 3; ++k) out[3 * m + k] = X[(i * 4 + j) * 3 + k];
  }
}

int64_t or_net_boundary(const double* ctrl, int64_t P, double* out_ctrl, int32_t* out_w) {
  edge_t* E = (edge_t*)malloc(sizeof(edge_t) * (size_t)(4 * P + 1));
  int64_t n = 0;
  for (int64_t p = 0; p < P; ++p) {
    for (int e = 0; e < 4; ++e) {
      double f[12], r[12];
      patch_edge(ctrl + 48 * p, e, f);
      for (int m = 0; m < 4; ++m)
        for (int k = 0; k < 3; ++k) r[3 * m + k] = f[3 * (3 - m) + k];
      int deg = 1;
      for (int k = 3; k < 12; ++k)
        if (f[k] != f[k % 3]) { deg = 0; break; }
      if (deg) continue;
      int c = cmp12(r, f);
      if (c < 0) { memcpy(E[n].c, r, sizeof r); E[n].w = -1; }
      else { memcpy(E[n].c, f, sizeof f); E[n].w = 1; }
      ++n;
    }
  }
  qsort(E, (size_t)n, sizeof(edge_t), cmp_edge);
  int64_t m = 0;
  for (int64_t i = 0; i < n;) {
    int64_t j = i;
    int32_t w = 0;
    while (j < n && cmp12(E[j].c, E[i].c) == 0) { w += E[j].w; ++j; }
    if (w != 0) {
      if (out_ctrl) {
        if (w > 0) memcpy(out_ctrl + 12 * m, E[i].c, sizeof(double) * 12);
        else
          for (int q = 0; q < 4; ++q)
            for (int k = 0; k < 3; ++k) out_ctrl[12 * m + 3 * q + k] = E[i].c[3 * (3 - q) + k];
      }
      if (out_w) out_w[m] = w > 0 ? w : -w;
      ++m;
    }
    i = j;
  }
  free(E);
  return m;
}

/* ------------------------------------------------------------------------- */
/* engine (retry policy SPEC.md:320,343,373-375,427)        */
/* ------------------------------------------------------------------------- */

typedef struct scene_t {
  const double* ctrl;
  int64_t P;
  double* lo;       /* (P,3) patch boxes */
  double* hi;
  int64_t n_edges;
  int S;
  double* verts;    /* (n_edges, S, 3) effective direction */
  int32_t* weight;
  double* band_h;   /* per edge sagitta bound */
  double diag;
  const or_params* prm;
} scene_t;

static void scene_build(scene_t* sc, const double* ctrl, int64_t P, const or_params* prm) {
  sc->ctrl = ctrl; sc->P = P; sc->prm = prm;
  sc->lo = (double*)malloc(sizeof(double) * 3 * (size_t)P);
  sc->hi = (double*)malloc(sizeof(double) * 3 * (size_t)P);
  double glo[3] = {INFINITY, INFINITY, INFINITY}, ghi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t p = 0; p < P; ++p) {
    aabb_of(ctrl + 48 * p, 16, sc->lo + 3 * p, sc->hi + 3 * p);
    for (int k = 0; k < 3; ++k) {
      glo[k] = fmin(glo[k], sc->lo[3 * p + k]);
      ghi[k] = fmax(ghi[k], sc->hi[3 * p + k]);
    }
  }
  double dg[3] = {ghi[0] - glo[0], ghi[1] - glo[1], ghi[2] - glo[2]};
  sc->diag = P > 0 ? norm3(dg) : 0.0;
  int64_t ne = or_net_boundary(ctrl, P, NULL, NULL);
  double* ec = (double*)malloc(sizeof(double) * 12 * (size_t)(ne + 1));
  sc->weight = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ne + 1));
  or_net_boundary(ctrl, P, ec, sc->weight);
  sc->n_edges = ne;
  sc->S = prm->samples_per_edge;
  sc->verts = (double*)malloc(sizeof(double) * 3 * (size_t)sc->S * (size_t)(ne + 1));
  sc->band_h = (double*)malloc(sizeof(double) * (size_t)(ne + 1));
  double dl = 1.0 / (double)(sc->S - 1);
  for (int64_t e = 0; e < ne; ++e) {
    const double* P4 = ec + 12 * e;
    or_sample_edge(P4, sc->S, sc->verts + (size_t)3 * sc->S * e);
    double m2 = 0.0;
    for (int q = 0; q < 2; ++q) {
      double s2[3];
      for (int k = 0; k < 3; ++k)
        s2[k] = P4[3 * (q + 2) + k] - 2.0 * P4[3 * (q + 1) + k] + P4[3 * q + k];
      m2 = fmax(m2, norm3(s2));
    }
    sc->band_h[e] = 0.75 * dl * dl * m2;   /* chord deviation <= D^2/8 * 6 max|2nd diff| */
  }
  free(ec);
}

static void scene_free(scene_t* sc) {
  free(sc->lo); free(sc->hi); free(sc->verts); free(sc->weight); free(sc->band_h);
}

/* one query, one direction: chi, boundary term, flags */
static void eval_dir(const scene_t* sc, const double p[3], const double d[3], int32_t* chi_out,
                     double* bterm_out, int32_t* flags_out) {
  const or_params* prm = sc->prm;
  int chi = 0, flags = 0;
  or_record rec[OR_MAX_ROOTS];
  for (int64_t q = 0; q < sc->P; ++q) {
    double c0, c1;
    if (!or_ray_aabb_clip(p, d, sc->lo + 3 * q, sc->hi + 3 * q, &c0, &c1)) continue;
    int n = or_patch_all_hits(sc->ctrl + 48 * q, p, d, prm, rec, OR_MAX_ROOTS);
    for (int i = 0; i < n; ++i) {
      chi += rec[i].sign;
      if (rec[i].tangency || rec[i].grazing) flags |= 1;
      if (fabs(rec[i].t) <= prm->on_surface_t) flags |= 4;
    }
  }
  double c[3] = {-d[0], -d[1], -d[2]};
  double total = 0.0;
  for (int64_t e = 0; e < sc->n_edges; ++e) {
    const double* V = sc->verts + (size_t)3 * sc->S * e;
    double s = 0.0;
    for (int k = 0; k + 1 < sc->S; ++k)
      s += fan_segment(V + 3 * k, V + 3 * (k + 1), p, c, prm->degenerate, sc->band_h[e], &flags,
                       prm->band_factor);
    total += (double)sc->weight[e] * s;
  }
  *chi_out = chi;
  *bterm_out = total / (4.0 * OR_PI);
  *flags_out = flags;
}

static void eval_query(const scene_t* sc, const double p0[3], int64_t qidx, double* w_out,
                       int8_t* st_out, int32_t* chi_out, int32_t* rounds_out) {
  const or_params* prm = sc->prm;
  double p[3] = {p0[0], p0[1], p0[2]};
  int jit = 0, jit_reason = 0, status = 2, r, used = 0;
  int32_t chi = 0, flags = 0;
  double bt = 0.0;
  for (r = 0; r < prm->max_rounds; ++r) {
    double d[3];
    or_direction(prm->dir_seed, r, d);
    eval_dir(sc, p, d, &chi, &bt, &flags);
    used = r + 1;
    if (flags & (4 | 8)) {                 /* on the surface / on the boundary: jitter */
      jit_reason = (flags & 4) ? 1 : 3;
      if (jit < prm->max_jitters) {
        ++jit;
        double v[3];
        or_jitter_dir(prm->dir_seed, qidx, jit, v);
        double s = prm->jitter_scale * sc->diag;
        for (int k = 0; k < 3; ++k) p[k] = p0[k] + s * v[k];
        continue;
      }
      status = 4;                          /* still on it after the jitter budget */
      break;
    }
    if (flags & (1 | 2)) continue;         /* tangent / grazing / band: new direction */
    status = jit ? jit_reason : 0;
    break;
  }
  *w_out = (double)chi + bt;
  *st_out = (int8_t)status;
  if (chi_out) *chi_out = chi;
  if (rounds_out) *rounds_out = used;
}

typedef struct job_t {
  const scene_t* sc;
  const double* queries;
  const int64_t* qidx;
  int64_t n;
  double* w;
  int8_t* st;
  int32_t* chi;
  int32_t* rounds;
  const double* dir;     /* non-NULL: eval_dir mode */
  double* bterm;
  int32_t* flags;
  int64_t next;
  pthread_mutex_t mu;
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t i0 = J->next;
    J->next += 16;
    pthread_mutex_unlock(&J->mu);
    if (i0 >= J->n) break;
    int64_t i1 = i0 + 16 < J->n ? i0 + 16 : J->n;
    for (int64_t i = i0; i < i1; ++i) {
      if (J->dir) {
        int32_t c, f;
        double b;
        eval_dir(J->sc, J->queries + 3 * i, J->dir, &c, &b, &f);
        J->chi[i] = c; J->bterm[i] = b; J->flags[i] = f;
      } else {
        eval_query(J->sc, J->queries + 3 * i, J->qidx ? J->qidx[i] : i, &J->w[i], &J->st[i],
                   J->chi ? &J->chi[i] : NULL, J->rounds ? &J->rounds[i] : NULL);
      }
    }
  }
  return NULL;
}

static void run_jobs(job_t* J, int nthreads) {
  if (nthreads <= 0) {
    nthreads = 1;
#ifdef _SC_NPROCESSORS_ONLN
    nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
#endif
  }
  if (nthreads > 256) nthreads = 256;
  pthread_mutex_init(&J->mu, NULL);
  J->next = 0;
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&J->mu);
}

int or_scene_eval(const double* ctrl, int64_t P, const double* queries, const int64_t* qidx,
                  int64_t n, const or_params* prm, double* w_out, int8_t* status_out,
                  int32_t* chi_out, int32_t* rounds_out, int nthreads) {
  if (prm->samples_per_edge < 2) return -1;
  scene_t sc;
  scene_build(&sc, ctrl, P, prm);
  job_t J;
  memset(&J, 0, sizeof J);
  J.sc = &sc; J.queries = queries; J.qidx = qidx; J.n = n;
  J.w = w_out; J.st = status_out; J.chi = chi_out; J.rounds = rounds_out;
  run_jobs(&J, nthreads);
  scene_free(&sc);
  return 0;
}

int or_scene_eval_dir(const double* ctrl, int64_t P, const double* queries, int64_t n,
                      const double d[3], const or_params* prm, int32_t* chi_out,
                      double* bterm_out, int32_t* flags_out, int nthreads) {
  if (prm->samples_per_edge < 2) return -1;
  scene_t sc;
  scene_build(&sc, ctrl, P, prm);
  job_t J;
  memset(&J, 0, sizeof J);
  J.sc = &sc; J.queries = queries; J.n = n;
  J.dir = d; J.chi = chi_out; J.bterm = bterm_out; J.flags = flags_out;
  run_jobs(&J, nthreads);
  scene_free(&sc);
  return 0;
}
