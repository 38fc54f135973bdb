/*
 * l1oracle.c -- CPU restatement of the reference GPSS path (TEST INFRASTRUCTURE ONLY).
 *
 * See l1oracle.h for scope and the reduction-order contract.  Build with
 *   gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math  (no -march: the reference's Release build
 *   targets baseline x86-64, which has no FMA, so every a*b+c rounds twice)
 * Every function cites the reference lines it follows (paths relative to
 * /root/reference/proj/core).
 */
#include "l1oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static int g_mode = ORC_CANONICAL;
void orc_set_mode(int mode) { g_mode = mode; }
int orc_get_mode(void) { return g_mode; }

/* ------------------------------------------------------------------------------------
 * Canonical pairwise summation.
 *
 * sum(t[0..m)) is the value of the complete binary tree over 2^ceil(log2 m) leaves whose
 * internal nodes are RN(left + right); leaves at index >= m are absent (a node with one
 * present child takes that child's value).  A binary counter evaluates the tree in one
 * left-to-right pass: lvl[l] holds the finished aligned block of 2^l leaves.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  double lvl[64];
  uint64_t count;
} pw_acc;

static inline void pw_init(pw_acc* a) { a->count = 0; }

static inline void pw_push(pw_acc* a, double v) {
  uint64_t i = a->count++;
  int l = 0;
  while (i & 1u) {
    v = a->lvl[l] + v;
    i >>= 1;
    ++l;
  }
  a->lvl[l] = v;
}

static inline double pw_final(const pw_acc* a) {
  uint64_t m = a->count;
  int have = 0;
  double acc = 0.0;
  for (int l = 0; m; ++l, m >>= 1) {
    if (m & 1u) {
      acc = have ? a->lvl[l] + acc : a->lvl[l];
      have = 1;
    }
  }
  return have ? acc : 0.0;
}

double orc_pairwise_sum(const double* t, int64_t m) {
  if (g_mode == ORC_LITERAL) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += t[i];
    return s;
  }
  pw_acc a;
  pw_init(&a);
  for (int64_t i = 0; i < m; ++i) pw_push(&a, t[i]);
  return pw_final(&a);
}

/* Eigen a.dot(b) / squaredNorm / lpNorm<1> / lpNorm<Infinity>: products are rounded, then
 * reduced in the active mode. */
double orc_dot(const double* a, const double* b, int64_t m) {
  if (g_mode == ORC_LITERAL) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += a[i] * b[i];
    return s;
  }
  pw_acc acc;
  pw_init(&acc);
  for (int64_t i = 0; i < m; ++i) pw_push(&acc, a[i] * b[i]);
  return pw_final(&acc);
}

double orc_sqnorm(const double* a, int64_t m) { return orc_dot(a, a, m); }

double orc_l1norm(const double* a, int64_t m) {
  if (g_mode == ORC_LITERAL) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += fabs(a[i]);
    return s;
  }
  pw_acc acc;
  pw_init(&acc);
  for (int64_t i = 0; i < m; ++i) pw_push(&acc, fabs(a[i]));
  return pw_final(&acc);
}

double orc_linf(const double* a, int64_t m) {
  double r = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double v = fabs(a[i]);
    if (v > r) r = v;
  }
  return r;
}

/* ------------------------------------------------------------------------------------
 * Dense operator.  linear_operator.hpp:45 (out = K x) and :46-48 (out = K^T r).
 * K is row-major n x p here; the reference stores Eigen column-major, which changes no
 * value because the reduction order is fixed by the mode, not by the storage.
 * ---------------------------------------------------------------------------------- */
/* OpenMP (when built with -fopenmp) splits the OUTPUTS across threads only: each output's
 * reduction runs in one thread in the order of the active mode, so the values do not depend
 * on the thread count (order-preserving; the full-size parity tests rely on this). */
void orc_apply(const double* K, int64_t n, int64_t p, const double* x, double* out) {
#pragma omp parallel for schedule(static) if (n * p > (1 << 18))
  for (int64_t i = 0; i < n; ++i) out[i] = orc_dot(K + i * p, x, p);
}

/* one block of columns [j0, j1) of K^T r; the carry pattern depends only on i */
static void adjoint_block(const double* K, int64_t n, int64_t p, const double* r, int64_t j0,
                          int64_t j1, double* out, double* lvl, double* cur, int levels) {
  const int64_t w = j1 - j0;
  if (g_mode == ORC_LITERAL) {
    for (int64_t j = 0; j < w; ++j) out[j0 + j] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double* row = K + i * p + j0;
      const double ri = r[i];
      for (int64_t j = 0; j < w; ++j) out[j0 + j] += row[j] * ri;
    }
    return;
  }
  (void)levels;
  for (int64_t i = 0; i < n; ++i) {
    const double* row = K + i * p + j0;
    const double ri = r[i];
    for (int64_t j = 0; j < w; ++j) cur[j] = row[j] * ri;
    uint64_t c = (uint64_t)i;
    int l = 0;
    while (c & 1u) {
      const double* lv = lvl + (size_t)l * (size_t)w;
      for (int64_t j = 0; j < w; ++j) cur[j] = lv[j] + cur[j];
      c >>= 1;
      ++l;
    }
    memcpy(lvl + (size_t)l * (size_t)w, cur, sizeof(double) * (size_t)w);
  }
  for (int64_t j = 0; j < w; ++j) out[j0 + j] = 0.0;
  uint64_t m = (uint64_t)n;
  int have = 0;
  for (int l = 0; m; ++l, m >>= 1) {
    if (m & 1u) {
      const double* lv = lvl + (size_t)l * (size_t)w;
      if (have)
        for (int64_t j = 0; j < w; ++j) out[j0 + j] = lv[j] + out[j0 + j];
      else
        memcpy(out + j0, lv, sizeof(double) * (size_t)w);
      have = 1;
    }
  }
}

/* per-column reductions over i (pairwise trees, or sequential in LITERAL mode), column
 * blocks split across threads */
void orc_apply_adjoint(const double* K, int64_t n, int64_t p, const double* r, double* out) {
  int levels = 1;
  while (((int64_t)1 << (levels - 1)) < n) ++levels;
  const int64_t bw = 512;
  const int64_t nb = (p + bw - 1) / bw;
#pragma omp parallel if (n * p > (1 << 18))
  {
    double* lvl = (double*)malloc(sizeof(double) * (size_t)levels * (size_t)bw);
    double* cur = (double*)malloc(sizeof(double) * (size_t)bw);
#pragma omp for schedule(static)
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t j0 = b * bw, j1 = j0 + bw < p ? j0 + bw : p;
      adjoint_block(K, n, p, r, j0, j1, out, lvl, cur, levels);
    }
    free(lvl);
    free(cur);
  }
}

/* linear_operator.cpp:43-60 */
int orc_spectral_norm(const double* K, int64_t n, int64_t p, int max_iters, double tol,
                      double* sigma_out, int64_t* matvecs) {
  if (max_iters < 1) return ORC_EINVAL;
  double* v = (double*)malloc(sizeof(double) * (size_t)p);
  double* kv = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)p);
  const double sq = sqrt((double)p);
  for (int64_t j = 0; j < p; ++j) v[j] = 1.0 / sq;
  double sigma = 0.0;
  int64_t mv = 0;
  int done = 0;
  for (int it = 0; it < max_iters; ++it) {
    orc_apply(K, n, p, v, kv);
    ++mv;
    const double sigma_new = sqrt(orc_sqnorm(kv, n));
    if (sigma_new == 0.0) {
      sigma = 0.0;
      done = 1;
      break;
    }
    orc_apply_adjoint(K, n, p, kv, w);
    ++mv;
    const double wn = sqrt(orc_sqnorm(w, p));
    for (int64_t j = 0; j < p; ++j) v[j] = w[j] / wn;
    if (it > 0 && fabs(sigma_new - sigma) <= tol * sigma_new) {
      sigma = sigma_new;
      done = 1;
      break;
    }
    sigma = sigma_new;
  }
  (void)done;
  *sigma_out = sigma;
  if (matvecs) *matvecs = mv;
  free(v);
  free(kv);
  free(w);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * prox.cpp
 * ---------------------------------------------------------------------------------- */
/* prox.cpp:23-36 (strict inequalities define the support) */
int orc_soft_threshold(const double* x, int64_t m, double t, double* out) {
  if (!(t >= 0.0)) return ORC_EINVAL;
  for (int64_t i = 0; i < m; ++i) {
    const double xi = x[i];
    if (xi > t)
      out[i] = xi - t;
    else if (xi < -t)
      out[i] = xi + t;
    else
      out[i] = 0.0;
  }
  return ORC_OK;
}

static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}

static int64_t count_nonzero(const double* a, int64_t m) {
  int64_t c = 0;
  for (int64_t i = 0; i < m; ++i) c += (a[i] != 0.0);
  return c;
}

/* prox.cpp:38-73 (project_l1_ball_with_threshold); prox.cpp:11-13 for rho < 0 */
int orc_project_l1(const double* x, int64_t m, double rho, double* out, double* theta_out,
                   int64_t* support) {
  if (!(rho >= 0.0)) return ORC_EINVAL;
  if (rho == 0.0) {
    for (int64_t i = 0; i < m; ++i) out[i] = 0.0;
    if (theta_out) *theta_out = orc_linf(x, m);
    if (support) *support = 0;
    return ORC_OK;
  }
  if (orc_l1norm(x, m) <= rho) {
    if (out != x) memcpy(out, x, sizeof(double) * (size_t)m);
    if (theta_out) *theta_out = 0.0;
    if (support) *support = count_nonzero(out, m);
    return ORC_OK;
  }
  double* mags = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) mags[i] = fabs(x[i]);
  qsort(mags, (size_t)m, sizeof(double), cmp_desc);
  double cumulative = 0.0, theta = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    cumulative += mags[i];
    const double candidate = (cumulative - rho) / (double)(i + 1);
    if (mags[i] > candidate)
      theta = candidate;
    else
      break;
  }
  free(mags);
  if (theta < 0.0) theta = 0.0;
  const double xinf = orc_linf(x, m);
  double* point = (double*)malloc(sizeof(double) * (size_t)m);
  orc_soft_threshold(x, m, theta, point);
  double bump = (theta > xinf ? theta : xinf) * DBL_EPSILON;
  int guard = 0;
  while (orc_l1norm(point, m) > rho && guard++ < 64) {
    theta += bump;
    bump *= 2.0;
    orc_soft_threshold(x, m, theta, point);
  }
  memcpy(out, point, sizeof(double) * (size_t)m);
  free(point);
  if (theta_out) *theta_out = theta;
  if (support) *support = count_nonzero(out, m);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * gpss.cpp
 * ---------------------------------------------------------------------------------- */
/* gpss.cpp:41-50 (plus this port's history cap of 64) */
int orc_config_validate(const orc_gp_config* c) {
  if (!(c->beta > 0.0 && c->beta < 1.0)) return ORC_EINVAL;
  if (!(c->theta > 0.0 && c->theta < 1.0)) return ORC_EINVAL;
  if (c->memory < 1 || c->memory > 64) return ORC_EINVAL;
  if (!(c->alpha_min > 0.0 && c->alpha_min < c->alpha_max)) return ORC_EINVAL;
  if (!(c->tau1 > 0.0 && c->tau1 < 1.0)) return ORC_EINVAL;
  if (c->alpha2_memory < 0 || c->alpha2_memory > 64) return ORC_EINVAL;
  return ORC_OK;
}

/* objective.cpp:42-48 */
int orc_stop_validate(const orc_stop_rule* s) {
  if (s->max_iterations <= 0 && s->max_matvecs <= 0 && s->max_seconds <= 0.0) return ORC_EINVAL;
  if (s->stationarity_tol < 0.0 || s->objective_tol < 0.0) return ORC_EINVAL;
  return ORC_OK;
}

/* gpss.cpp:18-20 */
double orc_clamp_step(double a, const orc_gp_config* cfg) {
  const double lo = a < cfg->alpha_max ? a : cfg->alpha_max; /* std::min(a, alpha_max) */
  return cfg->alpha_min > lo ? cfg->alpha_min : lo;          /* std::max(alpha_min, .) */
}

/* gpss.cpp:25-37 */
int orc_backtrack_quadratic(double f0, double a, double b, double f_max, double gd,
                            const orc_gp_config* cfg, double* step, double* f_new,
                            int* halvings) {
  double lam = 1.0;
  for (int h = 0; h <= 60; ++h) {
    const double f_trial = f0 + 2.0 * a * lam + b * lam * lam;
    if (f_trial <= f_max + cfg->beta * lam * gd) {
      *step = lam;
      *f_new = f_trial;
      *halvings = h;
      return ORC_OK;
    }
    lam *= cfg->theta;
  }
  return ORC_ERUNTIME;
}

/* gpss.cpp:52-57 */
void orc_steplength_init(orc_sl_state* st, const orc_gp_config* cfg) {
  st->tau = cfg->tau1;
  st->hist_len = 0;
}

/* gpss.cpp:59-91 on precomputed secant dots */
static void steplength_from_dots(orc_sl_state* st, double sz, double ss, double zz,
                                 const orc_gp_config* cfg, orc_sl_choice* c) {
  c->tau_before = st->tau;
  c->tau_after = st->tau;
  c->bb_active = 0;
  c->bb1_raw = NAN;
  c->bb2_raw = NAN;
  if (sz <= 0.0) {
    c->alpha = cfg->alpha_max;
    return;
  }
  c->bb_active = 1;
  c->bb1_raw = ss / sz;
  c->bb2_raw = sz / zz;
  const double a1 = orc_clamp_step(c->bb1_raw, cfg);
  const double a2 = orc_clamp_step(c->bb2_raw, cfg);
  st->hist[st->hist_len++] = a2;
  while (st->hist_len > cfg->alpha2_memory + 1) {
    memmove(st->hist, st->hist + 1, sizeof(double) * (size_t)(st->hist_len - 1));
    --st->hist_len;
  }
  if (a2 / a1 <= st->tau) {
    double mn = st->hist[0];
    for (int i = 1; i < st->hist_len; ++i)
      if (st->hist[i] < mn) mn = st->hist[i];
    c->alpha = mn;
    st->tau *= 0.9;
  } else {
    c->alpha = a1;
    st->tau *= 1.1;
  }
  c->tau_after = st->tau;
}

int orc_steplength_select(orc_sl_state* st, const double* s, const double* z, int64_t m,
                          const orc_gp_config* cfg, int64_t k, orc_sl_choice* out) {
  if (k < 1) return ORC_EINVAL;
  const double sz = orc_dot(s, z, m);
  double ss = 0.0, zz = 0.0;
  if (sz > 0.0) {
    ss = orc_dot(s, s, m);
    zz = orc_dot(z, z, m);
  }
  steplength_from_dots(st, sz, ss, zz, cfg, out);
  return ORC_OK;
}

/* gpss.cpp:93-98 */
double orc_alpha0_from_gradient(double rho, const double* x0, const double* grad, int64_t m,
                                const orc_gp_config* cfg) {
  double* v = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  for (int64_t i = 0; i < m; ++i) v[i] = x0[i] - grad[i];
  orc_project_l1(v, m, rho, v, NULL, NULL);
  const double norm = orc_linf(v, m);
  free(v);
  if (norm == 0.0) return cfg->alpha_max;
  return orc_clamp_step(1.0 / norm, cfg);
}

struct orc_gp {
  const double* K;
  int64_t n, p;
  const double* y;
  double rho;
  orc_gp_config cfg;
  double *x, *r, *g, *xp, *gp, *v, *h, *d, *kd;
  double f;
  int64_t k;
  double fh[64];
  int fh_len;
  double alpha0;
  int stationary;
  orc_sl_state sl;
  int64_t matvecs;
};

static double* dalloc(int64_t m) { return (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double)); }

void orc_gp_free(orc_gp* s) {
  if (!s) return;
  free(s->x); free(s->r); free(s->g); free(s->xp); free(s->gp);
  free(s->v); free(s->h); free(s->d); free(s->kd);
  free(s);
}

/* gpss.cpp:117-134 */
int orc_gp_init(const double* K, int64_t n, int64_t p, const double* y, double rho,
                const orc_gp_config* cfg, const double* x0, orc_gp** out) {
  *out = NULL;
  if (orc_config_validate(cfg)) return ORC_EINVAL;
  if (!(rho >= 0.0)) return ORC_EINVAL;
  orc_gp* s = (orc_gp*)calloc(1, sizeof(orc_gp));
  s->K = K; s->n = n; s->p = p; s->y = y; s->rho = rho; s->cfg = *cfg;
  s->x = dalloc(p); s->r = dalloc(n); s->g = dalloc(p); s->xp = dalloc(p); s->gp = dalloc(p);
  s->v = dalloc(p); s->h = dalloc(p); s->d = dalloc(p); s->kd = dalloc(n);
  if (x0) memcpy(s->x, x0, sizeof(double) * (size_t)p);
  if (!(orc_l1norm(s->x, p) <= rho + 1e-12)) { /* L1Ball::contains, prox.cpp:15-17 */
    orc_gp_free(s);
    return ORC_EINVAL;
  }
  orc_apply(K, n, p, s->x, s->r);
  ++s->matvecs;
  for (int64_t i = 0; i < n; ++i) s->r[i] = s->r[i] - y[i];
  s->f = orc_sqnorm(s->r, n);
  orc_apply_adjoint(K, n, p, s->r, s->g);
  ++s->matvecs;
  for (int64_t j = 0; j < p; ++j) s->g[j] = 2.0 * s->g[j];
  s->alpha0 = orc_alpha0_from_gradient(rho, s->x, s->g, p, cfg);
  s->fh[0] = s->f;
  s->fh_len = 1;
  orc_steplength_init(&s->sl, cfg);
  *out = s;
  return ORC_OK;
}

/* A caller writing GpIterationState's public fields (gpss.hpp:89-98) between steps, and
 * passing another GpConfig / L1Ball to gp_iterate (which takes both per call).  NULL vectors
 * are kept; SteplengthState (tau, history, prev_x, prev_grad) is kept. */
int orc_gp_set(orc_gp* s, const double* x, const double* r, const double* g, double f,
               int64_t k, const double* fh, int fh_len, const orc_gp_config* cfg, double rho) {
  if (fh_len < 1 || fh_len > 64 || k < 0) return ORC_EINVAL;
  if (cfg && orc_config_validate(cfg)) return ORC_EINVAL;
  if (x) memcpy(s->x, x, sizeof(double) * (size_t)s->p);
  if (r) memcpy(s->r, r, sizeof(double) * (size_t)s->n);
  if (g) memcpy(s->g, g, sizeof(double) * (size_t)s->p);
  s->f = f;
  s->k = k;
  memcpy(s->fh, fh, sizeof(double) * (size_t)fh_len);
  s->fh_len = fh_len;
  if (cfg) s->cfg = *cfg;
  s->rho = rho;
  return ORC_OK;
}

void orc_gp_get(const orc_gp* s, double* x, double* r, double* g, double* f, int64_t* k,
                double* alpha0, int64_t* matvecs) {
  if (x) memcpy(x, s->x, sizeof(double) * (size_t)s->p);
  if (r) memcpy(r, s->r, sizeof(double) * (size_t)s->n);
  if (g) memcpy(g, s->g, sizeof(double) * (size_t)s->p);
  if (f) *f = s->f;
  if (k) *k = s->k;
  if (alpha0) *alpha0 = s->alpha0;
  if (matvecs) *matvecs = s->matvecs;
}

/* gpss.cpp:136-219.  info receives the GpStepInfo fields in IterationRecord form. */
int orc_gp_iterate(orc_gp* s, double tol, orc_iter_record* info, int32_t* stationary) {
  const int64_t p = s->p, n = s->n;
  const orc_gp_config* cfg = &s->cfg;
  info->k = s->k;
  info->f = NAN; info->stationarity = NAN; info->alpha = NAN; info->step = NAN;
  info->bb_active = 0; info->halvings = 0;
  info->bb1_raw = NAN; info->bb2_raw = NAN; info->tau_before = NAN; info->tau_after = NAN;
  info->f_max = NAN; info->dir_derivative = NAN; info->theta = NAN; info->support = 0;
  *stationary = 0;
  if (s->stationary) {
    *stationary = 1;
    info->stationarity = 0.0;
    return ORC_OK;
  }
  /* Step 1: steplength (gpss.cpp:147-153) */
  double first_alpha;
  if (s->k == 0) {
    first_alpha = s->alpha0;
  } else {
    for (int64_t j = 0; j < p; ++j) {
      s->v[j] = s->x[j] - s->xp[j]; /* s */
      s->h[j] = s->g[j] - s->gp[j]; /* z */
    }
    orc_sl_choice c;
    orc_steplength_select(&s->sl, s->v, s->h, p, cfg, s->k, &c);
    first_alpha = c.alpha;
    info->bb_active = c.bb_active;
    info->bb1_raw = c.bb1_raw; info->bb2_raw = c.bb2_raw;
    info->tau_before = c.tau_before; info->tau_after = c.tau_after;
  }
  /* Steps 2-3: projection, direction and escalation (gpss.cpp:162-192) */
  double first_stat = 0.0, alpha = first_alpha;
  for (int first = 1;; first = 0) {
    for (int64_t j = 0; j < p; ++j) s->v[j] = s->x[j] - alpha * s->g[j];
    double theta;
    int64_t support;
    orc_project_l1(s->v, p, s->rho, s->h, &theta, &support);
    for (int64_t j = 0; j < p; ++j) s->d[j] = s->h[j] - s->x[j];
    const double stat = orc_linf(s->d, p);
    info->stationarity = stat;
    info->theta = theta;
    info->support = support;
    if (first) first_stat = stat;
    if (stat <= tol) {
      s->stationary = 1;
      *stationary = 1;
      info->alpha = alpha;
      info->f = s->f;
      return ORC_OK;
    }
    info->dir_derivative = orc_dot(s->g, s->d, p);
    if (info->dir_derivative < 0.0) break;
    if (alpha >= cfg->alpha_max) {
      s->stationary = 1;
      *stationary = 1;
      info->alpha = first_alpha;
      info->stationarity = first_stat;
      info->f = s->f;
      return ORC_OK;
    }
    alpha = (alpha * 10.0 < cfg->alpha_max) ? alpha * 10.0 : cfg->alpha_max;
  }
  info->alpha = alpha;
  /* forward product and line-search scalars (gpss.cpp:194-196) */
  orc_apply(s->K, n, p, s->d, s->kd);
  ++s->matvecs;
  const double a = orc_dot(s->r, s->kd, n);
  const double b = orc_sqnorm(s->kd, n);
  /* Steps 4-5 (gpss.cpp:199-203) */
  double f_max = s->fh[0];
  for (int i = 1; i < s->fh_len; ++i)
    if (s->fh[i] > f_max) f_max = s->fh[i];
  info->f_max = f_max;
  double step, f_new;
  int halvings;
  if (orc_backtrack_quadratic(s->f, a, b, f_max, info->dir_derivative, cfg, &step, &f_new,
                              &halvings))
    return ORC_ERUNTIME;
  info->step = step;
  info->halvings = halvings;
  /* Step 6 (gpss.cpp:206-215) */
  memcpy(s->xp, s->x, sizeof(double) * (size_t)p);
  memcpy(s->gp, s->g, sizeof(double) * (size_t)p);
  for (int64_t j = 0; j < p; ++j) s->x[j] = s->x[j] + step * s->d[j];
  for (int64_t i = 0; i < n; ++i) s->r[i] = s->r[i] + step * s->kd[i];
  s->f = f_new;
  orc_apply_adjoint(s->K, n, p, s->r, s->g);
  ++s->matvecs;
  for (int64_t j = 0; j < p; ++j) s->g[j] = 2.0 * s->g[j];
  s->fh[s->fh_len++] = s->f;
  while (s->fh_len > cfg->memory) {
    memmove(s->fh, s->fh + 1, sizeof(double) * (size_t)(s->fh_len - 1));
    --s->fh_len;
  }
  ++s->k;
  info->f = s->f;
  return ORC_OK;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* gpss.cpp:221-292 */
int orc_gpss_solve(const double* K, int64_t n, int64_t p, const double* y, double rho,
                   const orc_gp_config* cfg, const orc_stop_rule* stop, const double* x0,
                   double* x_out, orc_result* res, orc_iter_record* trace, int64_t trace_cap,
                   double* x_trace) {
  memset(res, 0, sizeof(*res));
  if (orc_stop_validate(stop)) return (res->status = ORC_EINVAL);
  const double t0 = now_seconds();
  orc_gp* s;
  int rc = orc_gp_init(K, n, p, y, rho, cfg, x0, &s);
  if (rc) return (res->status = rc);
  res->reason = ORC_MAX_ITERATIONS;
  res->objective = s->f;
  res->stationarity = INFINITY;
  double f_prev = s->f;
  for (int64_t k = 0;; ++k) {
    if (stop->max_iterations > 0 && k >= stop->max_iterations) {
      res->reason = ORC_MAX_ITERATIONS;
      break;
    }
    if (stop->max_matvecs > 0 && s->matvecs >= stop->max_matvecs) {
      res->reason = ORC_MAX_MATVECS;
      break;
    }
    if (stop->max_seconds > 0.0 && now_seconds() - t0 >= stop->max_seconds) {
      res->reason = ORC_MAX_SECONDS;
      break;
    }
    orc_iter_record info;
    int32_t stationary;
    rc = orc_gp_iterate(s, stop->stationarity_tol, &info, &stationary);
    if (rc) {
      orc_gp_free(s);
      return (res->status = rc);
    }
    res->stationarity = info.stationarity;
    if (stationary) {
      res->reason = ORC_STATIONARY;
      break;
    }
    res->iterations = s->k;
    res->objective = s->f;
    res->elapsed_seconds = now_seconds() - t0;
    if (trace && k < trace_cap) {
      info.k = k;
      info.matvecs = s->matvecs;
      info.elapsed_seconds = res->elapsed_seconds;
      trace[k] = info;
    }
    if (x_trace && k < trace_cap) memcpy(x_trace + k * p, s->x, sizeof(double) * (size_t)p);
    if (stop->objective_tol > 0.0 &&
        fabs(f_prev - s->f) <= stop->objective_tol * (fabs(s->f) > 1.0 ? fabs(s->f) : 1.0)) {
      res->reason = ORC_OBJECTIVE_TOL;
      break;
    }
    f_prev = s->f;
  }
  memcpy(x_out, s->x, sizeof(double) * (size_t)p);
  res->iterations = s->k;
  res->objective = s->f;
  res->matvecs = s->matvecs;
  res->f_history_len = s->fh_len;
  memcpy(res->f_history, s->fh, sizeof(double) * (size_t)s->fh_len);
  res->elapsed_seconds = now_seconds() - t0;
  orc_gp_free(s);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * Harness generators.  The reference draws problems from std::mt19937_64 + libm Box-Muller
 * (generators.cpp:13-26, rng.hpp:14-40); the BASELINE configs instead need on-device
 * generation of up to 8.6e9 entries, so both sides use a counter-based Philox4x32-10
 * stream and a normal transform built only from IEEE basic operations (+ - * / sqrt),
 * which the CUDA generator reproduces bit-for-bit.
 * ---------------------------------------------------------------------------------- */
void orc_philox4x32(uint32_t c[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t k0 = key[0], k1 = key[1];
  uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    x0 = hi1 ^ x1 ^ k0;
    x1 = lo1;
    x2 = hi0 ^ x3 ^ k1;
    x3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static inline double u53(uint32_t hi, uint32_t lo) {
  const uint64_t v = ((uint64_t)hi << 32) | lo;
  return (double)(v >> 11) * 0x1.0p-53;
}

/* log(u) for u in [2^-53, 1]: exact exponent split plus the atanh series on [1/sqrt2, sqrt2) */
double orc_det_log(double u) {
  uint64_t bits;
  memcpy(&bits, &u, 8);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  bits = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &bits, 8);
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double q = 1.0 / 25.0;
  q = q * s2 + 1.0 / 23.0;
  q = q * s2 + 1.0 / 21.0;
  q = q * s2 + 1.0 / 19.0;
  q = q * s2 + 1.0 / 17.0;
  q = q * s2 + 1.0 / 15.0;
  q = q * s2 + 1.0 / 13.0;
  q = q * s2 + 1.0 / 11.0;
  q = q * s2 + 1.0 / 9.0;
  q = q * s2 + 1.0 / 7.0;
  q = q * s2 + 1.0 / 5.0;
  q = q * s2 + 1.0 / 3.0;
  const double logm = 2.0 * s + 2.0 * s * (s2 * q);
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  return (double)e * ln2_hi + ((double)e * ln2_lo + logm);
}

/* sin(2 pi u), cos(2 pi u) for u in [0, 1): quadrant split, Taylor on [-pi/4, pi/4] */
void orc_det_sincos2pi(double u, double* so, double* co) {
  const double fq = floor(4.0 * u + 0.5);
  const int q = (int)fq;
  const double r = u - fq * 0.25;
  const double t = r * 6.283185307179586;
  const double t2 = t * t;
  double ps = -1.0 / 121645100408832000.0;           /* -1/19! */
  ps = ps * t2 + 1.0 / 355687428096000.0;             /* 1/17! */
  ps = ps * t2 - 1.0 / 1307674368000.0;               /* 1/15! */
  ps = ps * t2 + 1.0 / 6227020800.0;                  /* 1/13! */
  ps = ps * t2 - 1.0 / 39916800.0;                    /* 1/11! */
  ps = ps * t2 + 1.0 / 362880.0;                      /* 1/9! */
  ps = ps * t2 - 1.0 / 5040.0;
  ps = ps * t2 + 1.0 / 120.0;
  ps = ps * t2 - 1.0 / 6.0;
  const double sn = t + t * (t2 * ps);
  double pc = 1.0 / 6402373705728000.0;               /* 1/18! */
  pc = pc * t2 - 1.0 / 20922789888000.0;              /* 1/16! */
  pc = pc * t2 + 1.0 / 87178291200.0;                 /* 1/14! */
  pc = pc * t2 - 1.0 / 479001600.0;                   /* 1/12! */
  pc = pc * t2 + 1.0 / 3628800.0;                     /* 1/10! */
  pc = pc * t2 - 1.0 / 40320.0;
  pc = pc * t2 + 1.0 / 720.0;
  pc = pc * t2 - 1.0 / 24.0;
  pc = pc * t2 + 0.5;
  const double cs = 1.0 - t2 * pc;
  switch (q & 3) {
    case 0: *so = sn; *co = cs; break;
    case 1: *so = cs; *co = -sn; break;
    case 2: *so = -sn; *co = -cs; break;
    default: *so = -cs; *co = sn; break;
  }
}

double orc_uniform(uint64_t seed, uint32_t stream, uint64_t index) {
  uint32_t c[4] = {(uint32_t)index, (uint32_t)(index >> 32), stream, 0x5555u};
  const uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  orc_philox4x32(c, k, o);
  return u53(o[0], o[1]);
}

static void normal_pair(uint64_t seed, uint32_t stream, uint64_t pair, double* z0, double* z1) {
  uint32_t c[4] = {(uint32_t)pair, (uint32_t)(pair >> 32), stream, 0u};
  const uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  orc_philox4x32(c, k, o);
  const double u1 = 1.0 - u53(o[0], o[1]); /* (0, 1] */
  const double u2 = u53(o[2], o[3]);       /* [0, 1) */
  const double radius = sqrt(-2.0 * orc_det_log(u1));
  double sn, cs;
  orc_det_sincos2pi(u2, &sn, &cs);
  *z0 = radius * cs;
  *z1 = radius * sn;
}

double orc_normal(uint64_t seed, uint32_t stream, uint64_t index) {
  double z0, z1;
  normal_pair(seed, stream, index >> 1, &z0, &z1);
  return (index & 1u) ? z1 : z0;
}

void orc_fill_normal(uint64_t seed, uint32_t stream, uint64_t first, int64_t count,
                     double* out) {
#pragma omp parallel for schedule(static) if (count > (1 << 16))
  for (int64_t t = 0; t < count; ++t) out[t] = orc_normal(seed, stream, first + (uint64_t)t);
}

/* entry (i, j) is normal number i*p + j of stream 0 */
void orc_gaussian_matrix(uint64_t seed, int64_t n, int64_t p, double* K) {
  const uint64_t total = (uint64_t)n * (uint64_t)p;
  const int64_t pairs = (int64_t)(total / 2);
#pragma omp parallel for schedule(static) if (pairs > (1 << 16))
  for (int64_t q = 0; q < pairs; ++q)
    normal_pair(seed, 0u, (uint64_t)q, &K[2 * q], &K[2 * q + 1]);
  if (total & 1u) K[total - 1] = orc_normal(seed, 0u, total - 1);
}

/* square Toeplitz blur: K[i][j] = taps[i - j + radius] for |i - j| <= radius, else 0 */
void orc_blur_matrix(int64_t n, const double* taps, int radius, double* K) {
#pragma omp parallel for schedule(static) if (n > 1024)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t o = i - j;
      K[i * n + j] = (o >= -radius && o <= radius) ? taps[o + radius] : 0.0;
    }
}

void orc_scale(double* a, int64_t m, double c) {
#pragma omp parallel for schedule(static) if (m > (1 << 20))
  for (int64_t i = 0; i < m; ++i) a[i] = a[i] * c;
}

/* partial Fisher-Yates (rng.hpp:33-34 / generators.cpp:51-62 pattern) on a Philox stream */
int orc_sample_support(uint64_t seed, uint32_t stream, int64_t p, int64_t k, int64_t* idx) {
  if (k < 0 || k > p) return ORC_EINVAL;
  int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p > 0 ? p : 1));
  for (int64_t i = 0; i < p; ++i) pool[i] = i;
  for (int64_t t = 0; t < k; ++t) {
    const double u = orc_uniform(seed, stream, (uint64_t)t);
    int64_t j = t + (int64_t)floor(u * (double)(p - t));
    if (j >= p) j = p - 1;
    const int64_t tmp = pool[t];
    pool[t] = pool[j];
    pool[j] = tmp;
  }
  memcpy(idx, pool, sizeof(int64_t) * (size_t)k);
  free(pool);
  return ORC_OK;
}

/* ======================================================================== PSD, ISTA, FISTA */
/* f_history of these solvers keeps the newest 10 values (psd.cpp:68, shrinkage.cpp:33-36) */
static void hist_push10(orc_result* res, double f) {
  if (res->f_history_len < 10) {
    res->f_history[res->f_history_len++] = f;
  } else {
    for (int i = 0; i + 1 < 10; ++i) res->f_history[i] = res->f_history[i + 1];
    res->f_history[9] = f;
  }
}

/* budget checks at the top of an iteration (psd.cpp:24-35, shrinkage.cpp:16-31) */
static int budget_stop(const orc_stop_rule* stop, int64_t k, int64_t matvecs, double elapsed,
                       int32_t* reason) {
  if (stop->max_iterations > 0 && k >= stop->max_iterations) {
    *reason = ORC_MAX_ITERATIONS;
    return 1;
  }
  if (stop->max_matvecs > 0 && matvecs >= stop->max_matvecs) {
    *reason = ORC_MAX_MATVECS;
    return 1;
  }
  if (stop->max_seconds > 0.0 && elapsed >= stop->max_seconds) {
    *reason = ORC_MAX_SECONDS;
    return 1;
  }
  return 0;
}

/* ||a - b||_inf of two vectors (element differences first, as the Eigen expression) */
static double linf_diff(const double* a, const double* b, int64_t m, double* tmp) {
  for (int64_t i = 0; i < m; ++i) tmp[i] = a[i] - b[i];
  return orc_linf(tmp, m);
}

int orc_psd_solve(const double* K, int64_t n, int64_t p, const double* y, double rho,
                  const orc_stop_rule* stop, double* x_out, orc_result* res,
                  orc_iter_record* trace, int64_t trace_cap) {
  memset(res, 0, sizeof(*res));
  if (orc_stop_validate(stop)) return (res->status = ORC_EINVAL);
  if (!(rho >= 0.0)) return (res->status = ORC_EINVAL);
  const double t0 = now_seconds();
  double *x = dalloc(p), *xn = dalloc(p), *v = dalloc(p), *r = dalloc(p), *tmp = dalloc(p);
  double *kx = dalloc(n), *mis = dalloc(n), *kr = dalloc(n);
  int64_t mv = 0;
  double f_prev = INFINITY;
  res->reason = ORC_MAX_ITERATIONS;
  res->objective = NAN;
  res->stationarity = INFINITY;
  for (int64_t k = 0;; ++k) {
    if (budget_stop(stop, k, mv, now_seconds() - t0, &res->reason)) break;
    orc_apply(K, n, p, x, kx);  /* misfit = y - K x */
    ++mv;
    for (int64_t i = 0; i < n; ++i) mis[i] = y[i] - kx[i];
    const double f = orc_sqnorm(mis, n);
    orc_apply_adjoint(K, n, p, mis, r);
    ++mv;
    if (orc_linf(r, p) == 0.0) {
      res->objective = f;
      res->stationarity = 0.0;
      res->reason = ORC_STATIONARY;
      break;
    }
    orc_apply(K, n, p, r, kr);
    ++mv;
    const double denom = orc_sqnorm(kr, n);
    if (denom == 0.0) {
      res->objective = f;
      res->stationarity = 0.0;
      res->reason = ORC_STATIONARY;
      break;
    }
    const double beta = orc_sqnorm(r, p) / denom; /* exact line-search step */
    for (int64_t j = 0; j < p; ++j) v[j] = x[j] + beta * r[j];
    double th;
    int64_t sup;
    orc_project_l1(v, p, rho, xn, &th, &sup);
    const double stat = linf_diff(xn, x, p, tmp);
    memcpy(x, xn, sizeof(double) * (size_t)p);
    res->iterations = k + 1;
    res->objective = f;
    res->stationarity = stat;
    res->elapsed_seconds = now_seconds() - t0;
    hist_push10(res, f);
    if (trace && k < trace_cap) {
      orc_iter_record* t = &trace[k];
      memset(t, 0, sizeof(*t));
      t->k = k;
      t->f = f;
      t->stationarity = stat;
      t->alpha = beta;
      t->step = 1.0;
      t->matvecs = mv;
      t->elapsed_seconds = res->elapsed_seconds;
      t->theta = th;
      t->support = sup;
    }
    if (stop->stationarity_tol > 0.0 && stat <= stop->stationarity_tol) {
      res->reason = ORC_STATIONARY;
      break;
    }
    if (stop->objective_tol > 0.0 &&
        fabs(f_prev - f) <= stop->objective_tol * (fabs(f) > 1.0 ? fabs(f) : 1.0)) {
      res->reason = ORC_OBJECTIVE_TOL;
      break;
    }
    f_prev = f;
  }
  res->matvecs = mv;
  res->elapsed_seconds = now_seconds() - t0;
  memcpy(x_out, x, sizeof(double) * (size_t)p);
  free(x); free(xn); free(v); free(r); free(tmp); free(kx); free(mis); free(kr);
  return ORC_OK;
}

int orc_shrinkage_solve(const double* K, int64_t n, int64_t p, const double* y, double lambda,
                        int accelerated, const orc_stop_rule* stop, double* x_out,
                        orc_result* res, orc_iter_record* trace, int64_t trace_cap) {
  memset(res, 0, sizeof(*res));
  if (orc_stop_validate(stop)) return (res->status = ORC_EINVAL);
  if (!(lambda >= 0.0)) return (res->status = ORC_EINVAL); /* PenaltyWeight, prox.cpp */
  const double t0 = now_seconds();
  const double c = 0.999; /* kShrinkageOperatorScale, solver.hpp:128 */
  const double c2 = c * c;
  const double lam_eff = lambda * c2;
  double *x = dalloc(p), *xprev = dalloc(p), *pt = dalloc(p), *r = dalloc(p), *v = dalloc(p);
  double *xn = dalloc(p), *tmp = dalloc(p), *kp = dalloc(n), *mis = dalloc(n);
  int64_t mv = 0;
  double t = 1.0, f_prev = INFINITY;
  res->reason = ORC_MAX_ITERATIONS;
  res->objective = NAN;
  res->stationarity = INFINITY;
  for (int64_t k = 0;; ++k) {
    if (budget_stop(stop, k, mv, now_seconds() - t0, &res->reason)) break;
    memcpy(pt, x, sizeof(double) * (size_t)p);
    double t_next = t;
    if (accelerated) {
      t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)); /* fista_t_next, solver.hpp:118 */
      const double coef = (t - 1.0) / t_next;
      for (int64_t j = 0; j < p; ++j) pt[j] += coef * (x[j] - xprev[j]);
    }
    orc_apply(K, n, p, pt, kp);  /* misfit = K point - y */
    ++mv;
    for (int64_t i = 0; i < n; ++i) mis[i] = kp[i] - y[i];
    const double f = orc_sqnorm(mis, n);
    orc_apply_adjoint(K, n, p, mis, r);
    ++mv;
    for (int64_t j = 0; j < p; ++j) v[j] = pt[j] - c2 * r[j];
    orc_soft_threshold(v, p, lam_eff, xn);
    const double stat = linf_diff(xn, pt, p, tmp);
    memcpy(xprev, x, sizeof(double) * (size_t)p);
    memcpy(x, xn, sizeof(double) * (size_t)p);
    t = t_next;
    res->iterations = k + 1;
    res->objective = f;
    res->stationarity = stat;
    res->elapsed_seconds = now_seconds() - t0;
    hist_push10(res, f);
    if (trace && k < trace_cap) {
      orc_iter_record* tr = &trace[k];
      memset(tr, 0, sizeof(*tr));
      tr->k = k;
      tr->f = f;
      tr->stationarity = stat;
      tr->alpha = 1.0;
      tr->step = 1.0;
      tr->matvecs = mv;
      tr->elapsed_seconds = res->elapsed_seconds;
    }
    if (stop->stationarity_tol > 0.0 && stat <= stop->stationarity_tol) {
      res->reason = ORC_STATIONARY;
      break;
    }
    if (stop->objective_tol > 0.0 &&
        fabs(f_prev - f) <= stop->objective_tol * (fabs(f) > 1.0 ? fabs(f) : 1.0)) {
      res->reason = ORC_OBJECTIVE_TOL;
      break;
    }
    f_prev = f;
  }
  res->matvecs = mv;
  res->elapsed_seconds = now_seconds() - t0;
  memcpy(x_out, x, sizeof(double) * (size_t)p);
  free(x); free(xprev); free(pt); free(r); free(v); free(xn); free(tmp); free(kp); free(mis);
  return ORC_OK;
}

/* reference.cpp:9-13: ||x - S_lambda(x + K^T (y - K x))||_inf (2 matvecs) */
double orc_penalized_fpr(const double* K, int64_t n, int64_t p, const double* y,
                         const double* x, double lambda) {
  double *kx = dalloc(n), *mis = dalloc(n), *r = dalloc(p), *v = dalloc(p), *u = dalloc(p);
  double *tmp = dalloc(p);
  orc_apply(K, n, p, x, kx);
  for (int64_t i = 0; i < n; ++i) mis[i] = y[i] - kx[i];
  orc_apply_adjoint(K, n, p, mis, r);
  for (int64_t j = 0; j < p; ++j) v[j] = x[j] + r[j];
  orc_soft_threshold(v, p, lambda, u);
  const double c = linf_diff(x, u, p, tmp);
  free(kx); free(mis); free(r); free(v); free(u); free(tmp);
  return c;
}

/* reference.cpp:38-82: accelerated thresholding from x = 0 until the fixed-point certificate
 * holds (checked every check_interval iterations, or when the step is already below the
 * tolerance); lambda >= lambda_max gives the zero vector.  iters_out = iterations run. */
int orc_reference_minimizer(const double* K, int64_t n, int64_t p, const double* y,
                            double lambda, double oracle_tol, int64_t max_iterations,
                            int64_t check_interval, double* x_out, double* certificate,
                            int64_t* iters_out) {
  if (!(lambda > 0.0)) return ORC_EINVAL;
  double* g = dalloc(p);
  orc_apply_adjoint(K, n, p, y, g); /* lambda_max = ||K^T y||_inf (prox.cpp lambda_max) */
  const double lmax = orc_linf(g, p);
  free(g);
  memset(x_out, 0, sizeof(double) * (size_t)p);
  *iters_out = 0;
  if (lambda >= lmax) {
    *certificate = orc_penalized_fpr(K, n, p, y, x_out, lambda);
    return ORC_OK;
  }
  const double c = 0.999, c2 = c * c, lam_eff = lambda * c2; /* solver.hpp:128 */
  double *x = dalloc(p), *xprev = dalloc(p), *pt = dalloc(p), *r = dalloc(p), *v = dalloc(p);
  double *xn = dalloc(p), *tmp = dalloc(p), *kp = dalloc(n), *mis = dalloc(n);
  double t = 1.0;
  int rc = ORC_ERUNTIME;
  for (int64_t k = 0; k < max_iterations; ++k) {
    const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)); /* fista_t_next */
    const double coef = (t - 1.0) / t_next;
    for (int64_t j = 0; j < p; ++j) pt[j] = x[j] + coef * (x[j] - xprev[j]);
    orc_apply(K, n, p, pt, kp);
    for (int64_t i = 0; i < n; ++i) mis[i] = kp[i] - y[i];
    orc_apply_adjoint(K, n, p, mis, r);
    for (int64_t j = 0; j < p; ++j) v[j] = pt[j] - c2 * r[j];
    orc_soft_threshold(v, p, lam_eff, xn);
    memcpy(xprev, x, sizeof(double) * (size_t)p);
    memcpy(x, xn, sizeof(double) * (size_t)p);
    t = t_next;
    *iters_out = k + 1;
    const double surrogate = linf_diff(x, pt, p, tmp);
    if ((k + 1) % check_interval == 0 || surrogate <= oracle_tol) {
      const double cert = orc_penalized_fpr(K, n, p, y, x, lambda);
      if (cert <= oracle_tol) {
        *certificate = cert;
        rc = ORC_OK;
        break;
      }
    }
  }
  if (rc != ORC_OK) *certificate = orc_penalized_fpr(K, n, p, y, x, lambda);
  memcpy(x_out, x, sizeof(double) * (size_t)p);
  free(x); free(xprev); free(pt); free(r); free(v); free(xn); free(tmp); free(kp); free(mis);
  return rc;
}

/* ======================================================================== L1PROBv1 hash */
/* problem_io.cpp:115-125: FNV-1a 64 (offset basis 1469598103934665603, prime 1099511628211) */
uint64_t orc_fnv1a(const void* data, int64_t bytes, uint64_t h) {
  const unsigned char* c = (const unsigned char*)data;
  for (int64_t i = 0; i < bytes; ++i) {
    h ^= c[i];
    h *= 1099511628211ull;
  }
  return h;
}
