// C entry points into the reference's own solver sources (TEST INFRASTRUCTURE ONLY).
//
// oracle/build_ref.sh compiles this file together with the UNMODIFIED reference sources
// /root/reference/proj/core/src/{gpss,prox,linear_operator,objective,psd,shrinkage}.cpp
// against the
// Eigen stand-in in oracle/eigen_shim, producing oracle/_ref/libref_canon.so (canonical
// reductions, parity) and oracle/_ref/libref_fast.so (OpenMP GEMVs, CPU timing baseline).
// Structs are layout-compatible with oracle/l1oracle.h.
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>

#include "../oracle/l1oracle.h"
#include "l1solve/gpss.hpp"
#include "l1solve/prox.hpp"
#include "l1solve/problem_io.hpp"
#include "l1solve/reference.hpp"
#include "l1solve/solver.hpp"

using namespace l1solve;

namespace {
Matrix from_row_major(const double* K, long n, long p) {
  Matrix m(n, p);
  // blocked transpose into the column-major storage (OpenMP builds split the column tiles)
#pragma omp parallel for schedule(static) if (n * p > (1L << 20))
  for (long j0 = 0; j0 < p; j0 += 64)
    for (long i0 = 0; i0 < n; i0 += 64)
      for (long j = j0; j < std::min(j0 + 64, p); ++j)
        for (long i = i0; i < std::min(i0 + 64, n); ++i) m(i, j) = K[i * p + j];
  return m;
}
Vector vec(const double* x, long m) {
  Vector v(m);
  if (m) std::memcpy(v.data(), x, sizeof(double) * static_cast<size_t>(m));
  return v;
}
GpConfig conv(const orc_gp_config* c) {
  GpConfig g;
  g.beta = c->beta;
  g.theta = c->theta;
  g.memory = c->memory;
  g.alpha_min = c->alpha_min;
  g.alpha_max = c->alpha_max;
  g.tau1 = c->tau1;
  g.alpha2_memory = c->alpha2_memory;
  return g;
}
int code(const std::exception& e) {
  return dynamic_cast<const std::invalid_argument*>(&e) ? 1 : 2;
}
}  // namespace

struct ref_op {
  DenseOperator op;
};

extern "C" {

ref_op* ref_op_create(const double* K, long n, long p) {
  return new ref_op{DenseOperator(from_row_major(K, n, p))};
}
void ref_op_free(ref_op* o) { delete o; }

int ref_project_l1(const double* x, long m, double rho, double* out, double* theta) {
  try {
    const auto r = project_l1_ball_with_threshold(vec(x, m), L1Ball(rho));
    std::memcpy(out, r.point.data(), sizeof(double) * static_cast<size_t>(m));
    *theta = r.threshold;
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}

int ref_apply(ref_op* o, const double* x, double* out, int adjoint) {
  try {
    MatvecCounter mv;
    const long n = o->op.rows(), p = o->op.cols();
    if (adjoint) {
      const Vector r = o->op.apply_adjoint(vec(x, n), mv);
      std::memcpy(out, r.data(), sizeof(double) * static_cast<size_t>(p));
    } else {
      const Vector r = o->op.apply(vec(x, p), mv);
      std::memcpy(out, r.data(), sizeof(double) * static_cast<size_t>(n));
    }
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}

int ref_spectral_norm(ref_op* o, int max_iters, double tol, double* sigma) {
  try {
    *sigma = spectral_norm_estimate(o->op, max_iters, tol);
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}

int ref_gpss_solve(ref_op* o, const double* y, double rho, const orc_gp_config* cfg,
                   const orc_stop_rule* stop_in, const double* x0, double* x_out,
                   orc_result* res, orc_iter_record* trace, long trace_cap) {
  std::memset(res, 0, sizeof(*res));
  try {
    const long n = o->op.rows(), p = o->op.cols();
    const Objective obj(o->op, vec(y, n));
    StopRule stop;
    stop.max_iterations = stop_in->max_iterations;
    stop.max_matvecs = stop_in->max_matvecs;
    stop.max_seconds = stop_in->max_seconds;
    stop.stationarity_tol = stop_in->stationarity_tol;
    stop.objective_tol = stop_in->objective_tol;
    IterationCallback cb;
    if (trace && trace_cap > 0)
      cb = [&](const IterationRecord& r, const Vector&) {
        if (r.k >= trace_cap) return;
        orc_iter_record& t = trace[r.k];
        t.k = r.k;
        t.f = r.f;
        t.stationarity = r.stationarity;
        t.alpha = r.alpha;
        t.step = r.step;
        t.matvecs = r.matvecs;
        t.elapsed_seconds = r.elapsed_seconds;
        t.bb_active = r.bb_active;
        t.halvings = 0;
        t.bb1_raw = r.bb1_raw;
        t.bb2_raw = r.bb2_raw;
        t.tau_before = r.tau_before;
        t.tau_after = r.tau_after;
        t.f_max = r.f_max;
        t.dir_derivative = r.dir_derivative;
        t.theta = 0.0;
        t.support = 0;
      };
    const SolverState s = gpss_solve(obj, L1Ball(rho), conv(cfg), stop, cb,
                                     x0 ? vec(x0, p) : Vector());
    std::memcpy(x_out, s.x.data(), sizeof(double) * static_cast<size_t>(p));
    res->iterations = s.iterations;
    res->matvecs = s.matvecs.count;
    res->objective = s.objective;
    res->stationarity = s.stationarity;
    res->elapsed_seconds = s.elapsed_seconds;
    res->reason = static_cast<int>(s.reason);
    int i = 0;
    for (double f : s.f_history)
      if (i < 64) res->f_history[i++] = f;
    res->f_history_len = i;
    return 0;
  } catch (const std::exception& e) {
    return res->status = code(e);
  }
}

static StopRule conv_stop(const orc_stop_rule* s) {
  StopRule stop;
  stop.max_iterations = s->max_iterations;
  stop.max_matvecs = s->max_matvecs;
  stop.max_seconds = s->max_seconds;
  stop.stationarity_tol = s->stationarity_tol;
  stop.objective_tol = s->objective_tol;
  return stop;
}

static void fill_result(const SolverState& st, long p, double* x_out, orc_result* res) {
  std::memcpy(x_out, st.x.data(), sizeof(double) * static_cast<size_t>(p));
  res->iterations = st.iterations;
  res->matvecs = st.matvecs.count;
  res->objective = st.objective;
  res->stationarity = st.stationarity;
  res->elapsed_seconds = st.elapsed_seconds;
  res->reason = static_cast<int>(st.reason);
  int i = 0;
  for (double f : st.f_history)
    if (i < 64) res->f_history[i++] = f;
  res->f_history_len = i;
}

static IterationCallback record_cb(orc_iter_record* trace, long cap) {
  if (!trace || cap <= 0) return {};
  return [trace, cap](const IterationRecord& r, const Vector&) {
    if (r.k >= cap) return;
    orc_iter_record& t = trace[r.k];
    std::memset(&t, 0, sizeof(t));
    t.k = r.k;
    t.f = r.f;
    t.stationarity = r.stationarity;
    t.alpha = r.alpha;
    t.step = r.step;
    t.matvecs = r.matvecs;
    t.elapsed_seconds = r.elapsed_seconds;
  };
}

int ref_psd_solve(ref_op* o, const double* y, double rho, const orc_stop_rule* stop_in,
                  double* x_out, orc_result* res, orc_iter_record* trace, long trace_cap) {
  std::memset(res, 0, sizeof(*res));
  try {
    const Objective obj(o->op, vec(y, o->op.rows()));
    const SolverState s = psd_solve(obj, L1Ball(rho), conv_stop(stop_in), record_cb(trace, trace_cap));
    fill_result(s, o->op.cols(), x_out, res);
    return 0;
  } catch (const std::exception& e) {
    return res->status = code(e);
  }
}

int ref_shrinkage_solve(ref_op* o, const double* y, double lambda, int accelerated,
                        const orc_stop_rule* stop_in, double* x_out, orc_result* res,
                        orc_iter_record* trace, long trace_cap) {
  std::memset(res, 0, sizeof(*res));
  try {
    const Objective obj(o->op, vec(y, o->op.rows()));
    const auto cb = record_cb(trace, trace_cap);
    const SolverState s = accelerated
                              ? fista_solve(obj, PenaltyWeight(lambda), conv_stop(stop_in), cb)
                              : ista_solve(obj, PenaltyWeight(lambda), conv_stop(stop_in), cb);
    fill_result(s, o->op.cols(), x_out, res);
    return 0;
  } catch (const std::exception& e) {
    return res->status = code(e);
  }
}

static GeneratedProblem make_problem(const double* K, long n, long p, const double* y,
                                     const double* x_true, std::uint64_t seed, double noise) {
  GeneratedProblem g;
  g.op = std::make_shared<DenseOperator>(from_row_major(K, n, p));
  g.y = vec(y, n);
  g.x_true = vec(x_true, p);
  g.seed = seed;
  g.noise_level = noise;
  return g;
}

// problem_io.cpp: save / load / hash (L1PROBv1)
int ref_problem_save(const char* path, const double* K, long n, long p, const double* y,
                     const double* x_true, std::uint64_t seed, double noise) {
  try {
    save_problem(make_problem(K, n, p, y, x_true, seed, noise), path);
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}

int ref_problem_load(const char* path, long n, long p, double* K, double* y, double* x_true,
                     std::uint64_t* seed, double* noise) {
  try {
    const GeneratedProblem g = load_problem(path);
    const Matrix& m = g.op->matrix();
    if (m.rows() != n || m.cols() != p) return 1;
    for (long i = 0; i < n; ++i)
      for (long j = 0; j < p; ++j) K[i * p + j] = m(i, j);
    std::memcpy(y, g.y.data(), sizeof(double) * static_cast<size_t>(n));
    std::memcpy(x_true, g.x_true.data(), sizeof(double) * static_cast<size_t>(p));
    *seed = g.seed;
    *noise = g.noise_level;
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}

int ref_problem_hash(const double* K, long n, long p, const double* y, const double* x_true,
                     std::uint64_t seed, double noise, std::uint64_t* h) {
  try {
    *h = problem_hash(make_problem(K, n, p, y, x_true, seed, noise));
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}


int ref_reference_minimizer(ref_op* o, const double* y, double lambda, double oracle_tol,
                            long max_iterations, long check_interval, double* x_out,
                            double* certificate, double* rho, long* nnz) {
  try {
    const long n = o->op.rows(), p = o->op.cols();
    const Objective obj(o->op, vec(y, n));
    ReferenceOptions opt;
    opt.oracle_tol = oracle_tol;
    opt.max_iterations = max_iterations;
    opt.check_interval = check_interval;
    const ReferenceSolution r = reference_minimizer(obj, lambda, opt);
    std::memcpy(x_out, r.x.data(), sizeof(double) * static_cast<size_t>(p));
    *certificate = r.certificate;
    *rho = r.rho;
    *nnz = r.nnz;
    return 0;
  } catch (const std::exception& e) {
    return code(e);
  }
}
}  // extern "C"
