/*
 * l1g.h -- C-ABI of the B200-native GPSS engine (libl1g.so).
 *
 * This is the drop-in boundary for the reference solver path of l1solve
 * (/root/reference/proj/core).  Plain pointers and sizes only; every host pointer is a
 * caller-owned array of doubles, every device pointer a CUDA global-memory address on
 * the context's device.  Status codes mirror the reference's exception classes:
 *   L1G_OK (0), L1G_EINVAL (1) = std::invalid_argument, L1G_ERUNTIME (2) =
 *   std::runtime_error (CUDA failures, backtracking cap), L1G_ECANCELED (3) = an iteration
 *   callback asked to stop (its exception, in the C++ drop-in).  l1g_last_error() returns the
 *   thread's last message.
 *
 * Entry point -> reference interface it replaces (paths under proj/core):
 *   l1g_op_create_dense / l1g_op_destroy  -> DenseOperator(Matrix)      linear_operator.hpp:36-52
 *   l1g_op_apply / l1g_op_apply_adjoint   -> LinearOperator::apply /
 *                                             apply_adjoint (+1 matvec)  linear_operator.cpp:19-29
 *   l1g_op_spectral_norm                  -> spectral_norm_estimate     linear_operator.cpp:43-60
 *   l1g_project_l1                        -> project_l1_ball_with_threshold prox.cpp:38-73
 *   l1g_soft_threshold                    -> soft_threshold             prox.cpp:23-36
 *   l1g_steplength_select                 -> steplength_select          gpss.cpp:59-91
 *   l1g_backtrack                         -> backtracking_search core   gpss.cpp:25-37
 *   l1g_alpha0_from_gradient              -> alpha0_from_gradient       gpss.cpp:93-98
 *   l1g_solver_create / l1g_solver_init   -> gp_init                    gpss.cpp:117-134
 *   l1g_solver_iterate                    -> gp_iterate                 gpss.cpp:136-219
 *   l1g_gpss_solve / l1g_solver_run       -> gpss_solve                 gpss.cpp:221-292
 *   l1g_config_validate / l1g_stop_validate -> GpConfig::validate / StopRule::validate
 *                                                                        gpss.cpp:41-50,
 *                                                                        objective.cpp:42-48
 * Harness (BASELINE configs, not part of the reference API):
 *   l1g_op_generate_gaussian / l1g_op_generate_blur / l1g_op_scale / l1g_op_download.
 */
#ifndef L1G_H
#define L1G_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { L1G_OK = 0, L1G_EINVAL = 1, L1G_ERUNTIME = 2, L1G_ECANCELED = 3 };

/* StopReason, solver.hpp:38-44 */
enum { L1G_STATIONARY = 0, L1G_MAX_ITERATIONS = 1, L1G_MAX_MATVECS = 2, L1G_MAX_SECONDS = 3,
       L1G_OBJECTIVE_TOL = 4 };

typedef struct l1g_ctx l1g_ctx;
typedef struct l1g_op l1g_op;
typedef struct l1g_solver l1g_solver;

/* GpConfig, gpss.hpp:14-24 (memory and alpha2_memory are capped at 64 here) */
typedef struct {
  double beta, theta;
  int32_t memory, alpha2_memory;
  double alpha_min, alpha_max, tau1;
} l1g_gp_config;

/* StopRule, solver.hpp:52-60 */
typedef struct {
  int64_t max_iterations, max_matvecs;
  double max_seconds, stationarity_tol, objective_tol;
} l1g_stop_rule;

/* IterationRecord, solver.hpp:68-84, plus halvings, projection threshold and support */
typedef struct {
  int64_t k;
  double f, stationarity, alpha, step;
  int64_t matvecs;
  double elapsed_seconds;
  int32_t bb_active, halvings;
  double bb1_raw, bb2_raw, tau_before, tau_after, f_max, dir_derivative;
  double theta;
  int64_t support;
} l1g_iter_record;

/* SolverState scalars, solver.hpp:91-100 */
typedef struct {
  int64_t iterations, matvecs;
  double objective, stationarity, elapsed_seconds;
  int32_t reason, status;
  double f_history[64];
  int32_t f_history_len;
} l1g_result;

/* SteplengthState (gpss.hpp:31-36) without the cached vectors, and SteplengthChoice */
typedef struct {
  double tau;
  double hist[66];
  int32_t hist_len;
} l1g_sl_state;

typedef struct {
  double alpha;
  int32_t bb_active;
  double bb1_raw, bb2_raw, tau_before, tau_after;
} l1g_sl_choice;

const char* l1g_last_error(void);
const char* l1g_version(void);

/* ---- context ---- */
int l1g_ctx_create(int device, l1g_ctx** out);
void l1g_ctx_destroy(l1g_ctx* ctx);
int l1g_ctx_info(l1g_ctx* ctx, int* sm_count, int64_t* free_bytes);

/* ---- operator (device-resident tiled K) ---- */
int l1g_op_create_dense(l1g_ctx* ctx, const double* K, int64_t n, int64_t p, int row_major,
                        l1g_op** out);
int l1g_op_generate_gaussian(l1g_ctx* ctx, int64_t n, int64_t p, uint64_t seed,
                             int64_t col_offset, int64_t p_total, l1g_op** out);
int l1g_op_generate_blur(l1g_ctx* ctx, int64_t n, const double* taps, int radius,
                         l1g_op** out);
int l1g_op_scale(l1g_op* op, double c);
int l1g_op_dims(const l1g_op* op, int64_t* n, int64_t* p);
int l1g_op_download(l1g_op* op, double* K_row_major);
void l1g_op_destroy(l1g_op* op);

int l1g_op_apply(l1g_op* op, const double* x, double* out);
int l1g_op_apply_adjoint(l1g_op* op, const double* r, double* out);
/* device-pointer forms; stream may be NULL (legacy default stream of the context) */
int l1g_op_apply_dev(l1g_op* op, const double* x_dev, double* out_dev, void* stream);
int l1g_op_apply_adjoint_dev(l1g_op* op, const double* r_dev, double* out_dev, void* stream);
/* batched products on the FP64 tensor cores (mma.sync f64): X is B x p, R is B x n,
 * problem-major; results Y (B x n), G (B x p).  Accumulation order is the tensor core's,
 * so these agree with l1g_op_apply to rounding (not bit for bit). */
int l1g_op_apply_batched(l1g_op* op, int B, const double* X, double* Y);
int l1g_op_apply_adjoint_batched(l1g_op* op, int B, const double* R, double* G);
int l1g_op_spectral_norm(l1g_op* op, int max_iters, double tol, double* sigma,
                         int64_t* matvecs);

/* ---- prox ---- */
int l1g_project_l1(l1g_ctx* ctx, const double* x, int64_t m, double rho, double* out,
                   double* theta, int64_t* support);
int l1g_soft_threshold(l1g_ctx* ctx, const double* x, int64_t m, double t, double* out);
/* canonical reductions of host vectors: op 0 = a'b, 1 = ||a||^2, 2 = ||a||_1, 3 = ||a||_inf
 * (the Eigen dot / squaredNorm / lpNorm<1> / lpNorm<Infinity> the reference calls) */
int l1g_reduce(l1g_ctx* ctx, const double* a, const double* b, int64_t m, int op, double* out);

/* ---- GPSS pieces ---- */
int l1g_config_validate(const l1g_gp_config* cfg);
int l1g_stop_validate(const l1g_stop_rule* stop);
void l1g_steplength_init(l1g_sl_state* st, const l1g_gp_config* cfg);
int l1g_steplength_select(l1g_ctx* ctx, l1g_sl_state* st, const double* s, const double* z,
                          int64_t m, const l1g_gp_config* cfg, int64_t k, l1g_sl_choice* out);
int l1g_backtrack(l1g_ctx* ctx, double f0, double a, double b, double f_max, double gd,
                  const l1g_gp_config* cfg, double* step, double* f_new, int32_t* halvings);
int l1g_alpha0_from_gradient(l1g_ctx* ctx, double rho, const double* x0, const double* grad,
                             int64_t m, const l1g_gp_config* cfg, double* alpha0);

/* ---- solver (device-resident state) ---- */
int l1g_solver_create(l1g_op* op, const double* y, double rho, const l1g_gp_config* cfg,
                      l1g_solver** out);
int l1g_solver_set_y(l1g_solver* s, const double* y);
int l1g_solver_set_y_dev(l1g_solver* s, const double* y_dev);
int l1g_solver_init(l1g_solver* s, const double* x0 /* NULL = zero */);
int l1g_solver_iterate(l1g_solver* s, double stationarity_tol, l1g_iter_record* info,
                       int32_t* stationary);
int l1g_solver_run(l1g_solver* s, const l1g_stop_rule* stop, l1g_result* res,
                   l1g_iter_record* trace, int64_t trace_cap);
/* gpss_solve with an IterationCallback (solver.hpp:86-88): cb(record, x, p, user) after
 * every completed iteration; x is valid only during the call.  A nonzero return stops the
 * run at once and the call returns L1G_ECANCELED (the reference propagates a callback's
 * exception out of gpss_solve immediately; the C++ drop-in rethrows it). */
typedef int (*l1g_iter_cb)(const l1g_iter_record* rec, const double* x, int64_t p, void* user);
int l1g_solver_run_cb(l1g_solver* s, const l1g_stop_rule* stop, l1g_result* res,
                      l1g_iter_cb cb, void* user);
int l1g_solver_get(l1g_solver* s, double* x, double* kx_minus_y, double* grad, double* f,
                   int64_t* k, double* alpha0, int64_t* matvecs);
int l1g_solver_x_dev(l1g_solver* s, const double** x_dev);
/* The whole gp_iterate state (GpIterationState gpss.hpp:89-98 + SteplengthState :31-36), for
 * the drop-in's public-field GpIterationState: read it after gp_init / gp_iterate, write back
 * what a caller changed.  `choice` is the last steplength choice before any alpha escalation
 * (gpss.cpp:148-153); x_prev / grad_prev are SteplengthState::prev_x / prev_grad (valid when
 * has_prev, i.e. after the first step).  In set_state every vector may be NULL (kept); new
 * x / grad / x_prev / grad_prev recompute the secant dots s'z, s's, z'z on the device. */
typedef struct {
  double f;
  int64_t k;
  double alpha0;
  int32_t stationary, has_prev;
  int32_t f_history_len;
  double f_history[64];
  double tau;
  int32_t alpha2_len;
  double alpha2_history[66];
  l1g_sl_choice choice;
} l1g_gp_state;
int l1g_solver_get_state(l1g_solver* s, l1g_gp_state* st, double* x, double* kx_minus_y,
                         double* grad, double* x_prev, double* grad_prev);
int l1g_solver_set_state(l1g_solver* s, const l1g_gp_state* st, const double* x,
                         const double* kx_minus_y, const double* grad, const double* x_prev,
                         const double* grad_prev);
/* the GpConfig and L1Ball radius the next gp_iterate uses (gp_iterate takes both per call) */
int l1g_solver_set_problem(l1g_solver* s, const l1g_gp_config* cfg, double rho);

int l1g_solver_stream(l1g_solver* s, void** stream);
/* per-kernel CUDA-event timing of the device loop (projection / forward / adjoint), summed
 * over completed iterations, and the number of kernels this solver launched */
int l1g_solver_set_timing(l1g_solver* s, int on);
/* ---- L1PROBv1 problem files (problem_io.cpp, docs/problem_format.md):
 *   l1g_problem_info  -> header of a file (n, p, seed, noise_level)
 *   l1g_problem_load  -> load_problem: K streamed into a new device operator; y (n) and
 *                        x_true (p) into caller buffers (either may be NULL)
 *   l1g_problem_save  -> save_problem (K read back from the device)
 *   l1g_problem_hash  -> problem_hash: FNV-1a 64 of the serialized bytes */
int l1g_problem_info(const char* path, int64_t* n, int64_t* p, uint64_t* seed, double* noise);
int l1g_problem_load(l1g_ctx* ctx, const char* path, double* y, double* x_true, uint64_t* seed,
                     double* noise, l1g_op** out);
int l1g_problem_save(const char* path, l1g_op* op, const double* y, const double* x_true,
                     uint64_t seed, double noise);
int l1g_problem_hash(l1g_op* op, const double* y, const double* x_true, uint64_t seed,
                     double noise, uint64_t* hash);

/* ---- the reference's other solvers of the problem family, on the same
 * device kernels; trace may be NULL.  x0 = 0 as in the reference.
 *   l1g_psd_solve       -> psd_solve    psd.cpp:14-93  (projected steepest descent)
 *   l1g_shrinkage_solve -> ista_solve / fista_solve (accelerated = 1) shrinkage.cpp:41-118 */
int l1g_psd_solve(l1g_op* op, const double* y, double rho, const l1g_stop_rule* stop,
                  double* x_out, l1g_result* res, l1g_iter_record* trace, int64_t cap,
                  l1g_iter_cb cb, void* user);
int l1g_shrinkage_solve(l1g_op* op, const double* y, double lambda, int accelerated,
                        const l1g_stop_rule* stop, double* x_out, l1g_result* res,
                        l1g_iter_record* trace, int64_t cap, l1g_iter_cb cb, void* user);

/* ---- the reference minimizer of the penalized problem (reference.cpp:38-82), on the
 * device FISTA kernels: accelerated thresholding from x = 0 until the fixed-point certificate
 * ||x - S_lambda(x + K^T (y - K x))||_inf <= oracle_tol (checked every check_interval
 * iterations, or once a step is below the tolerance).  opt NULL = ReferenceOptions defaults
 * (1e-12, 500000, 50, 1e-10).  Not converged: L1G_ERUNTIME (as the reference throws).
 *   l1g_penalized_fixed_point_residual -> penalized_fixed_point_residual reference.cpp:9-13 */
typedef struct {
  double oracle_tol;
  int64_t max_iterations, check_interval;
  double nnz_threshold;
} l1g_ref_options;
typedef struct {
  double lambda, rho, oracle_tol, certificate;
  int64_t nnz, iterations, matvecs;
} l1g_ref_solution;
int l1g_reference_minimizer(l1g_op* op, const double* y, double lambda,
                            const l1g_ref_options* opt, double* x_out, l1g_ref_solution* out);
int l1g_penalized_fixed_point_residual(l1g_op* op, const double* y, const double* x,
                                       double lambda, double* out);

/* ---- column-sharded runs (no reference counterpart: the reference is
 * single-threaded).  Shard r of R holds columns [r*p/R, (r+1)*p/R) of K as its own l1g_op
 * (p/R a multiple of 256) and owns that slice of x and g.  Each iteration exchanges the shard
 * tree values of K d (n doubles per shard) and, after the adjoint, the shard's packet: its new
 * x and g slices and its subtree values of s'z, s's, z'z with its clock (2 p/R + 8 doubles);
 * the projection runs on the gathered x, g and joins the dots over the ranks.  With p/R a
 * power of two the result is bit-identical to the unsharded solve.
 *   l1g_solver_create_group: R shards in this process on one device, run in lockstep
 *     (exchange = device copies); the other l1g_solver_* calls take the returned leader.
 *   l1g_comm_*: an NCCL communicator, one shard per process (rank r owns shard r). */
typedef struct l1g_comm l1g_comm;
int l1g_solver_create_group(l1g_op* const* ops, int nshards, const double* y, double rho,
                            const l1g_gp_config* cfg, l1g_solver** out);
int l1g_comm_unique_id(void* id128);
int l1g_comm_create(l1g_ctx* ctx, int rank, int nranks, const void* id128, l1g_comm** out);
/* a communicator whose transport is the caller's own host allgather (no NCCL): every
 * exchange is staged through pinned host memory and `fn` runs as a host node of the
 * iteration graph -- e.g. gloo between processes sharing one GPU in tests.  fn must fill
 * recv[r * count + i] with rank r's send[i] and return 0. */
typedef int (*l1g_allgather_fn)(const double* send, double* recv, int64_t count, void* user);
int l1g_comm_create_host(l1g_ctx* ctx, int rank, int nranks, l1g_allgather_fn fn, void* user,
                         l1g_comm** out);
void l1g_comm_destroy(l1g_comm* comm);
int l1g_solver_create_sharded(l1g_op* op, l1g_comm* comm, const double* y, double rho,
                              const l1g_gp_config* cfg, l1g_solver** out);
/* average duration of the two per-iteration exchanges (K d values; [x | g | dots] packets) over `reps`
 * standalone launches on the solver stream (NCCL time, reported next to the solve) */
int l1g_solver_time_exchange(l1g_solver* s, int reps, double* kd_ms, double* g_ms);
/* ---- batched right-hand sides (BASELINE C5): B
 * problems sharing K, with their own y_b (Y is B x n, problem-major) and rho_b, solved in
 * lockstep.  Each problem follows gpss_solve (gpss.cpp:221-292) and counts its matvecs as if
 * solved alone; the products run on the FP64 tensor cores, so iterates agree with the
 * per-problem solve to rounding.  X0 / X are B x p. */
typedef struct l1g_batch l1g_batch;
int l1g_batch_create(l1g_op* op, int B, const double* Y, const double* rho,
                     const l1g_gp_config* cfg, l1g_batch** out);
int l1g_batch_init(l1g_batch* b, const double* X0);
int l1g_batch_run(l1g_batch* b, const l1g_stop_rule* stop, l1g_result* results);
/* continue after l1g_batch_run with a larger budget: problems a budget stopped resume
 * exactly where they stopped; stationary / objective-tol stops stay stopped (one trajectory
 * sampled at a budget ladder, isochrone.cpp:75-100) */
int l1g_batch_resume(l1g_batch* b, const l1g_stop_rule* stop, l1g_result* results);
int l1g_batch_get_x(l1g_batch* b, double* X);
int l1g_batch_stream(l1g_batch* b, void** stream);
int l1g_batch_launches(l1g_batch* b, int64_t* launches, int reset);
int l1g_batch_time_products(l1g_batch* b, int reps, double* fwd_ms, double* adj_ms);
void l1g_batch_destroy(l1g_batch* b);
int l1g_gpss_solve_batched(l1g_op* op, int B, const double* Y, const double* rho,
                           const l1g_gp_config* cfg, const l1g_stop_rule* stop, double* X_out,
                           l1g_result* results);
/* forward product of the iteration (gpss.cpp:194, DenseOperator::do_apply,
 * linear_operator.hpp:45-46), all modes giving the same bits:
 *   1 = over the columns where d != 0 only, switching on the device to the dense stream
 *       when d has at least L1G_FWD_DENSE_FRAC (default 0.8) * p nonzeros (default);
 *   2 = over the columns where d != 0 only, never switching;
 *   0 = dense streaming pass over all of K.
 * Environment L1G_FWD=dense / L1G_FWD=sparse set 0 / 2 at creation. */
int l1g_solver_set_forward(l1g_solver* s, int sparse);
/* 1 if the solver runs the step after the projection as the one-cluster small-problem kernel
 * (K within one cluster's shared memory: n_pad <= 384, p_pad <= 1024; L1G_SMALL=0 disables),
 * 0 if it runs the large path's four kernels */
int l1g_solver_small_path(l1g_solver* s, int* small);
/* projection phase profile accumulated since gp_init (32 doubles): [0..7] SM cycles per
 * phase, [8] calls, [9] attempts, [10] pivot rounds, [11] candidates, [12] bumps,
 * [13] retries, [14..17], [21], [22] sub-phases of the cluster sort, [18..19] sparse
 * forward support columns / calls, [20] prefix epochs, [23] forward products the density
 * switch ran as the dense stream, [24..30] sub-phases of the
 * cluster-wide exact prefix (CTA 0's SM cycles) */
int l1g_solver_proj_profile(l1g_solver* s, double* out32);
int l1g_solver_timing(l1g_solver* s, double* proj_ms, double* fwd_ms, double* adj_ms,
                      int64_t* iterations, int64_t* launches, int reset);
void l1g_solver_destroy(l1g_solver* s);

/* gpss_solve(Objective(op, y), L1Ball(rho), cfg, stop, {}, x0) */
int l1g_gpss_solve(l1g_op* op, const double* y, double rho, const l1g_gp_config* cfg,
                   const l1g_stop_rule* stop, const double* x0, double* x_out, l1g_result* res,
                   l1g_iter_record* trace, int64_t trace_cap);

/* harness random streams: kind 0 = standard normal #index, 1 = uniform [0,1) #index of the
 * Philox stream (seed, stream) -- bit-identical to oracle orc_normal / orc_uniform */
int l1g_rng_fill(l1g_ctx* ctx, int kind, uint64_t seed, uint32_t stream, uint64_t first,
                 int64_t count, double* out);

/* pinned host buffers for the end-to-end path */
int l1g_host_alloc(int64_t bytes, void** ptr);
void l1g_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif
