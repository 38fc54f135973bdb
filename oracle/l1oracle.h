/*
 * l1oracle.h -- CPU restatement of the reference GPSS path (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker for the B200 product in paper_0902_4424_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product never links or calls it.
 *
 * It restates, in plain C, the reference l1solve sources under /root/reference/proj/core:
 *   gpss.cpp:18-292  (clamp, backtrack_quadratic, steplength_select, alpha0, gp_init,
 *                     gp_iterate, gpss_solve)
 *   prox.cpp:11-77   (L1Ball::contains, soft_threshold, project_l1_ball_with_threshold)
 *   linear_operator.cpp:19-60, linear_operator.hpp:45-48 (dense apply / adjoint, power
 *                     iteration)
 *   objective.cpp:42-48 (StopRule::validate)
 *
 * Reduction order.  The reference delegates every dot product, norm and GEMV to Eigen,
 * whose summation order is an unspecified property of a third-party library that is
 * absent here.  The oracle therefore offers two reduction modes:
 *   ORC_CANONICAL (default): every sum is the *pairwise* sum with power-of-two splits
 *     (see orc_pairwise_sum) of correctly-rounded products (no FMA).  This is the
 *     reduction-order contract the CUDA kernels implement, so GPU and oracle agree
 *     bit-for-bit (up to the sign of zero).
 *   ORC_LITERAL: plain left-to-right sequential sums (the naive reading of the reference);
 *     used for tolerance-based comparisons.
 * Everything that the reference itself orders explicitly (the sorted sequential cumulative
 * sum in prox.cpp:43-52, the backtracking arithmetic in gpss.cpp:30-31, ...) is restated
 * operation for operation.
 */
#ifndef L1ORACLE_H
#define L1ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_CANONICAL = 0, ORC_LITERAL = 1 };

/* Stop reasons, solver.hpp:38-44 */
enum { ORC_STATIONARY = 0, ORC_MAX_ITERATIONS = 1, ORC_MAX_MATVECS = 2, ORC_MAX_SECONDS = 3,
       ORC_OBJECTIVE_TOL = 4 };

/* Status codes: 0 ok, 1 invalid_argument, 2 runtime_error (mirrors the C++ exceptions). */
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ERUNTIME = 2 };

typedef struct {
  double beta, theta;
  int32_t memory;
  int32_t alpha2_memory;
  double alpha_min, alpha_max, tau1;
} orc_gp_config; /* gpss.hpp:14-24 */

typedef struct {
  int64_t max_iterations;
  int64_t max_matvecs;
  double max_seconds, stationarity_tol, objective_tol;
} orc_stop_rule; /* solver.hpp:52-60 */

/* IterationRecord (solver.hpp:68-84) plus the projection threshold / support size and
 * the backtracking halvings of the accepted step. */
typedef struct {
  int64_t k;
  double f, stationarity, alpha, step;
  int64_t matvecs;
  double elapsed_seconds;
  int32_t bb_active, halvings;
  double bb1_raw, bb2_raw, tau_before, tau_after, f_max, dir_derivative;
  double theta;
  int64_t support;
} orc_iter_record;

typedef struct {
  int64_t iterations, matvecs;
  double objective, stationarity, elapsed_seconds;
  int32_t reason, status;
  double f_history[64];
  int32_t f_history_len;
} orc_result;

void orc_set_mode(int mode);
int orc_get_mode(void);

/* ---- reductions ---- */
double orc_pairwise_sum(const double* t, int64_t m);
double orc_dot(const double* a, const double* b, int64_t m);
double orc_sqnorm(const double* a, int64_t m);
double orc_l1norm(const double* a, int64_t m);
double orc_linf(const double* a, int64_t m);

/* ---- dense operator: K row-major n x p ---- */
void orc_apply(const double* K, int64_t n, int64_t p, const double* x, double* out);
void orc_apply_adjoint(const double* K, int64_t n, int64_t p, const double* r, double* out);
int orc_spectral_norm(const double* K, int64_t n, int64_t p, int max_iters, double tol,
                      double* sigma, int64_t* matvecs);

/* ---- prox ---- */
int orc_soft_threshold(const double* x, int64_t m, double t, double* out);
int orc_project_l1(const double* x, int64_t m, double rho, double* out, double* theta,
                   int64_t* support);

/* ---- GPSS pieces (gpss.cpp) ---- */
int orc_config_validate(const orc_gp_config* cfg);
int orc_stop_validate(const orc_stop_rule* stop);
double orc_clamp_step(double a, const orc_gp_config* cfg);
int orc_backtrack_quadratic(double f0, double a, double b, double f_max, double gd,
                            const orc_gp_config* cfg, double* step, double* f_new,
                            int* halvings);

typedef struct {
  double tau;
  double hist[66];
  int32_t hist_len;
} orc_sl_state;

typedef struct {
  double alpha;
  int32_t bb_active;
  double bb1_raw, bb2_raw, tau_before, tau_after;
} orc_sl_choice;

void orc_steplength_init(orc_sl_state* st, const orc_gp_config* cfg);
int orc_steplength_select(orc_sl_state* st, const double* s, const double* z, int64_t m,
                          const orc_gp_config* cfg, int64_t k, orc_sl_choice* out);
double orc_alpha0_from_gradient(double rho, const double* x0, const double* grad, int64_t m,
                                const orc_gp_config* cfg);

/* Full solver: gpss.cpp:221-292.  x0 may be NULL (zero start).  trace may be NULL. */
int orc_gpss_solve(const double* K, int64_t n, int64_t p, const double* y, double rho,
                   const orc_gp_config* cfg, const orc_stop_rule* stop, const double* x0,
                   double* x_out, orc_result* res, orc_iter_record* trace, int64_t trace_cap,
                   double* x_trace /* iterations x p, optional */);

/* Projected steepest descent, psd.cpp:14-93 (3 matvecs per iteration, x0 = 0). */
int orc_psd_solve(const double* K, int64_t n, int64_t p, const double* y, double rho,
                  const orc_stop_rule* stop, double* x_out, orc_result* res,
                  orc_iter_record* trace, int64_t trace_cap);
/* ISTA (accelerated = 0) / FISTA (accelerated = 1), shrinkage.cpp:41-118, on the rescaled
 * problem (c = 0.999, solver.hpp:128), x0 = 0. */
int orc_shrinkage_solve(const double* K, int64_t n, int64_t p, const double* y, double lambda,
                        int accelerated, const orc_stop_rule* stop, double* x_out,
                        orc_result* res, orc_iter_record* trace, int64_t trace_cap);

/* Stateful single-step interface (gp_init / gp_iterate) for step-level tests. */
typedef struct orc_gp orc_gp;
int orc_gp_init(const double* K, int64_t n, int64_t p, const double* y, double rho,
                const orc_gp_config* cfg, const double* x0, orc_gp** out);
int orc_gp_iterate(orc_gp* st, double stationarity_tol, orc_iter_record* info,
                   int32_t* stationary);
void orc_gp_get(const orc_gp* st, double* x, double* kx_minus_y, double* grad, double* f,
                int64_t* k, double* alpha0, int64_t* matvecs);
void orc_gp_free(orc_gp* st);
int orc_gp_set(orc_gp* st, const double* x, const double* kx_minus_y, const double* grad,
               double f, int64_t k, const double* f_history, int f_history_len,
               const orc_gp_config* cfg, double rho);

/* ---- reference.cpp:9-82: penalized fixed-point residual and the reference minimizer ---- */
double orc_penalized_fpr(const double* K, int64_t n, int64_t p, const double* y,
                         const double* x, double lambda);
int orc_reference_minimizer(const double* K, int64_t n, int64_t p, const double* y,
                            double lambda, double oracle_tol, int64_t max_iterations,
                            int64_t check_interval, double* x_out, double* certificate,
                            int64_t* iters_out);

/* ---- L1PROBv1 (problem_io.cpp): FNV-1a 64 over serialized bytes, chained from h */
uint64_t orc_fnv1a(const void* data, int64_t bytes, uint64_t h);

/* ---- harness generators (deterministic, bit-identical to the device generators) ---- */
void orc_philox4x32(uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double orc_det_log(double u);
void orc_det_sincos2pi(double u, double* s, double* c);
/* standard normal number `index` of stream (seed, stream); pairs come from Box-Muller */
double orc_normal(uint64_t seed, uint32_t stream, uint64_t index);
double orc_uniform(uint64_t seed, uint32_t stream, uint64_t index);
void orc_fill_normal(uint64_t seed, uint32_t stream, uint64_t first, int64_t count,
                     double* out);
void orc_gaussian_matrix(uint64_t seed, int64_t n, int64_t p, double* K /* row-major */);
void orc_blur_matrix(int64_t n, const double* taps, int radius, double* K);
void orc_scale(double* a, int64_t m, double c);
int orc_sample_support(uint64_t seed, uint32_t stream, int64_t p, int64_t k, int64_t* idx);

#ifdef __cplusplus
}
#endif
#endif
