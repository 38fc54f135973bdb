// l1solve_dropin.cpp -- the reference's C++ solver API (include/l1solve/*.hpp) on top of
// the C-ABI (include/l1g.h).  Builds into libl1solve_b200.so, linked against libl1g.so.
//
// DenseOperator problems run the device-resident loop (l1g_gpss_solve / l1g_solver_*); their
// GpIterationState mirrors the device state in the reference's public fields.  A
// user-defined LinearOperator (matrix-free K) keeps the reference's host-driven gp_init /
// gp_iterate / gpss_solve (gpss.cpp:117-292 restated below) with every reduction, the
// projection, the steplength rule and the backtracking executed by the same device code.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "l1g.h"
#include "l1solve/gpss.hpp"
#include "l1solve/generators.hpp"
#include "l1solve/problem_io.hpp"
#include "l1solve/reference.hpp"
#include "l1solve/rng.hpp"

namespace l1solve {

namespace {

void check(int rc) {
  if (rc == L1G_OK) return;
  const char* m = l1g_last_error();
  if (rc == L1G_EINVAL) throw std::invalid_argument(m ? m : "invalid argument");
  throw std::runtime_error(m ? m : "l1g runtime error");
}

l1g_ctx* ctx() {
  static std::once_flag once;
  static l1g_ctx* c = nullptr;
  std::call_once(once, [] {
    int dev = 0;
    if (const char* e = std::getenv("L1G_DEVICE")) dev = std::atoi(e);
    check(l1g_ctx_create(dev, &c));
  });
  return c;
}

double reduce(const Vector& a, const Vector* b, int op) {
  double out = 0.0;
  check(l1g_reduce(ctx(), a.data(), b ? b->data() : nullptr, a.size(), op, &out));
  return out;
}

l1g_gp_config conv(const GpConfig& c) {
  l1g_gp_config g;
  g.beta = c.beta;
  g.theta = c.theta;
  g.memory = c.memory;
  g.alpha2_memory = c.alpha2_memory;
  g.alpha_min = c.alpha_min;
  g.alpha_max = c.alpha_max;
  g.tau1 = c.tau1;
  return g;
}

l1g_stop_rule conv(const StopRule& s) {
  l1g_stop_rule r;
  r.max_iterations = s.max_iterations;
  r.max_matvecs = s.max_matvecs;
  r.max_seconds = s.max_seconds;
  r.stationarity_tol = s.stationarity_tol;
  r.objective_tol = s.objective_tol;
  return r;
}

IterationRecord conv(const l1g_iter_record& r) {
  IterationRecord o;
  o.k = r.k;
  o.f = r.f;
  o.stationarity = r.stationarity;
  o.alpha = r.alpha;
  o.step = r.step;
  o.matvecs = r.matvecs;
  o.elapsed_seconds = r.elapsed_seconds;
  o.bb_active = r.bb_active != 0;
  o.bb1_raw = r.bb1_raw;
  o.bb2_raw = r.bb2_raw;
  o.tau_before = r.tau_before;
  o.tau_after = r.tau_after;
  o.f_max = r.f_max;
  o.dir_derivative = r.dir_derivative;
  return o;
}

SolverState state_from(const l1g_result& r, Vector x) {
  SolverState s;
  s.x = std::move(x);
  s.iterations = r.iterations;
  s.matvecs.count = r.matvecs;
  for (int i = 0; i < r.f_history_len; ++i) s.f_history.push_back(r.f_history[i]);
  s.objective = r.objective;
  s.stationarity = r.stationarity;
  s.elapsed_seconds = r.elapsed_seconds;
  s.reason = static_cast<StopReason>(r.reason);
  return s;
}

[[noreturn]] void dim_error(const char* what, Index got, Index want) {
  throw std::invalid_argument(std::string(what) + ": vector has length " + std::to_string(got) +
                              ", operator expects " + std::to_string(want));
}

}  // namespace

// ------------------------------------------------------------------------- Vector
double Vector::dot(const Vector& o) const {
  if (o.size() != size()) throw std::invalid_argument("dot: size mismatch");
  return reduce(*this, &o, 0);
}
double Vector::squaredNorm() const { return reduce(*this, nullptr, 1); }
double Vector::norm() const { return std::sqrt(squaredNorm()); }
template <>
double Vector::lpNorm<1>() const {
  return reduce(*this, nullptr, 2);
}
template <>
double Vector::lpNorm<Infinity>() const {
  return reduce(*this, nullptr, 3);
}
// element-wise updates are single IEEE operations: identical wherever they run
Vector& Vector::operator+=(const Vector& o) {
  if (o.size() != size()) throw std::invalid_argument("+=: size mismatch");
  for (Index i = 0; i < size(); ++i) (*this)[i] = (*this)[i] + o[i];
  return *this;
}
Vector& Vector::operator-=(const Vector& o) {
  if (o.size() != size()) throw std::invalid_argument("-=: size mismatch");
  for (Index i = 0; i < size(); ++i) (*this)[i] = (*this)[i] - o[i];
  return *this;
}
Vector& Vector::operator*=(double c) {
  for (Index i = 0; i < size(); ++i) (*this)[i] = (*this)[i] * c;
  return *this;
}
Vector& Vector::operator/=(double c) {
  for (Index i = 0; i < size(); ++i) (*this)[i] = (*this)[i] / c;
  return *this;
}
Vector operator+(Vector a, const Vector& b) { return a += b; }
Vector operator-(Vector a, const Vector& b) { return a -= b; }
Vector operator-(Vector a) {
  for (Index i = 0; i < a.size(); ++i) a[i] = -a[i];
  return a;
}
Vector operator*(double c, Vector a) {
  for (Index i = 0; i < a.size(); ++i) a[i] = c * a[i];
  return a;
}
Vector operator*(Vector a, double c) { return a *= c; }
Vector operator/(Vector a, double c) { return a /= c; }

// ------------------------------------------------------------------------- operators
void LinearOperator::apply(const Vector& x, Vector& out, MatvecCounter& mv) const {
  if (x.size() != cols()) dim_error("apply", x.size(), cols());
  if (out.size() != rows()) out = Vector(rows());
  do_apply(x, out);
  ++mv.count;
}
void LinearOperator::apply_adjoint(const Vector& r, Vector& out, MatvecCounter& mv) const {
  if (r.size() != rows()) dim_error("apply_adjoint", r.size(), rows());
  if (out.size() != cols()) out = Vector(cols());
  do_apply_adjoint(r, out);
  ++mv.count;
}
Vector LinearOperator::apply(const Vector& x, MatvecCounter& mv) const {
  Vector out(rows());
  apply(x, out, mv);
  return out;
}
Vector LinearOperator::apply_adjoint(const Vector& r, MatvecCounter& mv) const {
  Vector out(cols());
  apply_adjoint(r, out, mv);
  return out;
}

DenseOperator::DenseOperator(const Matrix& k) : n_(k.rows()), p_(k.cols()) {
  check(l1g_op_create_dense(ctx(), k.data(), n_, p_, /*row_major=*/0, &op_));
}
DenseOperator::~DenseOperator() { l1g_op_destroy(op_); }
Matrix DenseOperator::matrix() const {
  std::vector<double> rm(static_cast<std::size_t>(n_ * p_));
  check(l1g_op_download(op_, rm.data()));
  Matrix m(n_, p_);
  for (Index i = 0; i < n_; ++i)
    for (Index j = 0; j < p_; ++j) m(i, j) = rm[static_cast<std::size_t>(i * p_ + j)];
  return m;
}
void DenseOperator::do_apply(const Vector& x, Vector& out) const {
  check(l1g_op_apply(op_, x.data(), out.data()));
}
void DenseOperator::do_apply_adjoint(const Vector& r, Vector& out) const {
  check(l1g_op_apply_adjoint(op_, r.data(), out.data()));
}

double spectral_norm_estimate(const LinearOperator& op, int max_iters, double tol,
                              MatvecCounter& mv) {
  if (max_iters < 1) throw std::invalid_argument("spectral_norm_estimate: max_iters must be >= 1");
  if (auto* d = dynamic_cast<const DenseOperator*>(&op)) {
    double s = 0.0;
    int64_t m = 0;
    check(l1g_op_spectral_norm(d->handle(), max_iters, tol, &s, &m));
    mv.count += m;
    return s;
  }
  // matrix-free operator: linear_operator.cpp:43-60 with device reductions
  const Index p = op.cols();
  Vector v = Vector::Ones(p) / std::sqrt(static_cast<double>(p));
  double sigma = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    const Vector kv = op.apply(v, mv);
    const double sn = kv.norm();
    if (sn == 0.0) return 0.0;
    const Vector w = op.apply_adjoint(kv, mv);
    v = w / w.norm();
    if (it > 0 && std::abs(sn - sigma) <= tol * sn) return sn;
    sigma = sn;
  }
  return sigma;
}
double spectral_norm_estimate(const LinearOperator& op, int max_iters, double tol) {
  MatvecCounter scratch;
  return spectral_norm_estimate(op, max_iters, tol, scratch);
}

// ------------------------------------------------------------------------- prox
L1Ball::L1Ball(double rho) : rho_(rho) {
  if (!(rho >= 0.0)) throw std::invalid_argument("L1Ball: radius must be >= 0");
}
bool L1Ball::contains(const Vector& x, double tol) const { return x.lpNorm<1>() <= rho_ + tol; }
PenaltyWeight::PenaltyWeight(double lambda) : lambda_(lambda) {
  if (!(lambda >= 0.0)) throw std::invalid_argument("PenaltyWeight: lambda must be >= 0");
}
Vector soft_threshold(const Vector& x, double t) {
  Vector out(x.size());
  check(l1g_soft_threshold(ctx(), x.data(), x.size(), t, out.data()));
  return out;
}
L1Projection project_l1_ball_with_threshold(const Vector& x, const L1Ball& ball) {
  L1Projection r{Vector(x.size()), 0.0};
  int64_t sup = 0;
  check(l1g_project_l1(ctx(), x.data(), x.size(), ball.radius(), r.point.data(), &r.threshold,
                       &sup));
  return r;
}
Vector project_l1_ball(const Vector& x, const L1Ball& ball) {
  return project_l1_ball_with_threshold(x, ball).point;
}
double lambda_max(const LinearOperator& op, const Vector& y, MatvecCounter& mv) {
  return op.apply_adjoint(y, mv).lpNorm<Infinity>();
}
double lambda_max(const LinearOperator& op, const Vector& y) {
  MatvecCounter s;
  return lambda_max(op, y, s);
}
double lambda_from_rho(const LinearOperator& op, const Vector& y, const Vector& x_rho,
                       MatvecCounter& mv) {
  const Vector misfit = y - op.apply(x_rho, mv);
  return op.apply_adjoint(misfit, mv).lpNorm<Infinity>();
}
double lambda_from_rho(const LinearOperator& op, const Vector& y, const Vector& x_rho) {
  MatvecCounter s;
  return lambda_from_rho(op, y, x_rho, s);
}
double rho_from_lambda(const Vector& x_lambda) { return x_lambda.lpNorm<1>(); }

// ------------------------------------------------------------------------- objective
Objective::Objective(const LinearOperator& op, Vector y) : op_(&op), y_(std::move(y)) {
  if (y_.size() != op_->rows())
    throw std::invalid_argument("Objective: data vector length does not match operator rows");
}
double Objective::value(const Vector& x, MatvecCounter& mv) const {
  return (op_->apply(x, mv) - y_).squaredNorm();
}
Vector Objective::residual(const Vector& x, MatvecCounter& mv) const {
  return op_->apply_adjoint(y_ - op_->apply(x, mv), mv);
}
Vector Objective::gradient(const Vector& x, MatvecCounter& mv) const {
  return -2.0 * residual(x, mv);
}
double Objective::value_and_gradient(const Vector& x, Vector& grad, MatvecCounter& mv) const {
  const Vector misfit = op_->apply(x, mv) - y_;
  grad = 2.0 * op_->apply_adjoint(misfit, mv);
  return misfit.squaredNorm();
}

std::string to_string(StopReason r) {
  switch (r) {
    case StopReason::Stationary: return "stationary";
    case StopReason::MaxIterations: return "max_iterations";
    case StopReason::MaxMatvecs: return "max_matvecs";
    case StopReason::MaxSeconds: return "max_seconds";
    case StopReason::ObjectiveTol: return "objective_tol";
  }
  return "unknown";
}

void StopRule::validate() const {
  const l1g_stop_rule s = conv(*this);
  check(l1g_stop_validate(&s));
}
void GpConfig::validate() const {
  const l1g_gp_config c = conv(*this);
  check(l1g_config_validate(&c));
}

// ------------------------------------------------------------------------- gpss pieces
SteplengthState steplength_init(const GpConfig& cfg) {
  cfg.validate();
  SteplengthState st;
  st.tau = cfg.tau1;
  return st;
}

SteplengthChoice steplength_select(SteplengthState& st, const Vector& s, const Vector& z,
                                   const GpConfig& cfg, long k) {
  if (s.size() != z.size()) throw std::invalid_argument("steplength_select: size mismatch");
  l1g_sl_state ds;
  std::memset(&ds, 0, sizeof(ds));
  ds.tau = st.tau;
  for (double h : st.alpha2_history) ds.hist[ds.hist_len++] = h;
  const l1g_gp_config c = conv(cfg);
  l1g_sl_choice ch;
  check(l1g_steplength_select(ctx(), &ds, s.data(), z.data(), s.size(), &c, k, &ch));
  st.tau = ds.tau;
  st.alpha2_history.assign(ds.hist, ds.hist + ds.hist_len);
  SteplengthChoice o;
  o.alpha = ch.alpha;
  o.bb_active = ch.bb_active != 0;
  o.bb1_raw = ch.bb1_raw;
  o.bb2_raw = ch.bb2_raw;
  o.tau_before = ch.tau_before;
  o.tau_after = ch.tau_after;
  return o;
}

double alpha0_from_gradient(const L1Ball& ball, const Vector& x0, const Vector& grad,
                            const GpConfig& cfg) {
  const l1g_gp_config c = conv(cfg);
  double a = 0.0;
  check(l1g_alpha0_from_gradient(ctx(), ball.radius(), x0.data(), grad.data(), x0.size(), &c, &a));
  return a;
}

double alpha0_init(const Objective& prob, const L1Ball& ball, const Vector& x0,
                   const GpConfig& cfg, MatvecCounter& mv) {
  cfg.validate();
  return alpha0_from_gradient(ball, x0, prob.gradient(x0, mv), cfg);
}

BacktrackResult backtracking_search(const Objective& prob, const Vector& x, const Vector& d,
                                    double f_max, double dir_derivative, const GpConfig& cfg,
                                    MatvecCounter& mv) {
  if (!(dir_derivative < 0.0))
    throw std::invalid_argument("backtracking_search: d must be a descent direction");
  const Vector misfit = prob.op().apply(x, mv) - prob.y();
  const Vector kd = prob.op().apply(d, mv);
  const l1g_gp_config c = conv(cfg);
  BacktrackResult r;
  int32_t h = 0;
  check(l1g_backtrack(ctx(), misfit.squaredNorm(), misfit.dot(kd), kd.squaredNorm(), f_max,
                      dir_derivative, &c, &r.step, &r.f_new, &h));
  r.halvings = h;
  return r;
}

// ------------------------------------------------------------------------- gp state
namespace detail {
// A DenseOperator problem's GpIterationState on the GPU (an l1g_solver) and the state the
// device last reported, against which the caller's fields are compared before each step.
struct DeviceIterationState {
  l1g_solver* s = nullptr;
  Index n = 0, p = 0;
  Vector x, r, g, x_prev, g_prev;
  double f = 0.0, alpha0 = 0.0, tau = 0.0, rho = 0.0;
  long k = 0;
  bool stationary = false, has_prev = false;
  std::deque<double> fh, a2h;
  GpConfig cfg;
  ~DeviceIterationState() { l1g_solver_destroy(s); }
};
}  // namespace detail

namespace {
using detail::DeviceIterationState;

bool bits_equal(const Vector& a, const Vector& b) {
  return a.size() == b.size() &&
         (a.size() == 0 ||
          std::memcmp(a.data(), b.data(), sizeof(double) * static_cast<std::size_t>(a.size())) == 0);
}
bool bits_equal(const std::deque<double>& a, const std::deque<double>& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (std::memcmp(&a[i], &b[i], sizeof(double)) != 0) return false;
  return true;
}
bool same_cfg(const GpConfig& a, const GpConfig& b) {
  return a.beta == b.beta && a.theta == b.theta && a.memory == b.memory &&
         a.alpha_min == b.alpha_min && a.alpha_max == b.alpha_max && a.tau1 == b.tau1 &&
         a.alpha2_memory == b.alpha2_memory;
}
int64_t solver_matvecs(l1g_solver* s) {
  int64_t mv = 0;
  check(l1g_solver_get(s, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &mv));
  return mv;
}
SteplengthChoice conv(const l1g_sl_choice& c) {
  SteplengthChoice o;
  o.alpha = c.alpha;
  o.bb_active = c.bb_active != 0;
  o.bb1_raw = c.bb1_raw;
  o.bb2_raw = c.bb2_raw;
  o.tau_before = c.tau_before;
  o.tau_after = c.tau_after;
  return o;
}

// device -> the caller's GpIterationState / SteplengthState (and the comparison copy)
l1g_gp_state pull(DeviceIterationState& d, GpIterationState& st, SteplengthState* sls) {
  l1g_gp_state g;
  d.x = Vector(d.p);
  d.r = Vector(d.n);
  d.g = Vector(d.p);
  d.x_prev = Vector(d.p);
  d.g_prev = Vector(d.p);
  check(l1g_solver_get_state(d.s, &g, d.x.data(), d.r.data(), d.g.data(), d.x_prev.data(),
                             d.g_prev.data()));
  d.f = g.f;
  d.k = static_cast<long>(g.k);
  d.alpha0 = g.alpha0;
  d.stationary = g.stationary != 0;
  d.has_prev = g.has_prev != 0;
  d.fh.assign(g.f_history, g.f_history + g.f_history_len);
  d.tau = g.tau;
  d.a2h.assign(g.alpha2_history, g.alpha2_history + g.alpha2_len);
  st.x = d.x;
  st.kx_minus_y = d.r;
  st.grad = d.g;
  st.f = d.f;
  st.k = d.k;
  st.f_history = d.fh;
  st.alpha0 = d.alpha0;
  st.stationary = d.stationary;
  if (sls) {
    sls->tau = d.tau;
    sls->alpha2_history = d.a2h;
    if (d.has_prev) {
      sls->prev_x = d.x_prev;
      sls->prev_grad = d.g_prev;
    }
  }
  return g;
}

// the caller's state, steplength state, GpConfig and ball -> device, where they differ from
// what the device last reported
void push(DeviceIterationState& d, const GpIterationState& st, const SteplengthState& sls,
          const GpConfig& cfg, const L1Ball& ball) {
  if (!same_cfg(cfg, d.cfg) || ball.radius() != d.rho) {
    const l1g_gp_config c = conv(cfg);
    check(l1g_solver_set_problem(d.s, &c, ball.radius()));
    d.cfg = cfg;
    d.rho = ball.radius();
  }
  if (st.x.size() != d.p || st.grad.size() != d.p || st.kx_minus_y.size() != d.n)
    throw std::invalid_argument("gp_iterate: state vectors do not match the operator");
  const double* x = bits_equal(st.x, d.x) ? nullptr : st.x.data();
  const double* r = bits_equal(st.kx_minus_y, d.r) ? nullptr : st.kx_minus_y.data();
  const double* g = bits_equal(st.grad, d.g) ? nullptr : st.grad.data();
  const bool prev = st.k > 0 && sls.prev_x.size() == d.p && sls.prev_grad.size() == d.p;
  const double* xp = prev && !(d.has_prev && bits_equal(sls.prev_x, d.x_prev)) ? sls.prev_x.data()
                                                                              : nullptr;
  const double* gp = prev && !(d.has_prev && bits_equal(sls.prev_grad, d.g_prev))
                         ? sls.prev_grad.data()
                         : nullptr;
  const bool scalars = st.f != d.f || st.k != d.k || !bits_equal(st.f_history, d.fh) ||
                       st.alpha0 != d.alpha0 || st.stationary != d.stationary ||
                       sls.tau != d.tau || !bits_equal(sls.alpha2_history, d.a2h);
  if (!scalars && !x && !r && !g && !xp && !gp) return;
  if (st.f_history.empty() || st.f_history.size() > 64 || sls.alpha2_history.size() > 66)
    throw std::invalid_argument("gp_iterate: history lengths out of range (at most 64)");
  l1g_gp_state in;
  std::memset(&in, 0, sizeof(in));
  in.f = st.f;
  in.k = st.k;
  in.alpha0 = st.alpha0;
  in.stationary = st.stationary;
  in.f_history_len = static_cast<int32_t>(st.f_history.size());
  std::copy(st.f_history.begin(), st.f_history.end(), in.f_history);
  in.tau = sls.tau;
  in.alpha2_len = static_cast<int32_t>(sls.alpha2_history.size());
  std::copy(sls.alpha2_history.begin(), sls.alpha2_history.end(), in.alpha2_history);
  check(l1g_solver_set_state(d.s, &in, x, r, g, xp, gp));
  d.x = st.x;
  d.r = st.kx_minus_y;
  d.g = st.grad;
  if (xp) d.x_prev = sls.prev_x;
  if (gp) d.g_prev = sls.prev_grad;
  d.has_prev = d.has_prev || prev;
  d.f = st.f;
  d.k = st.k;
  d.fh = st.f_history;
  d.alpha0 = st.alpha0;
  d.stationary = st.stationary;
  d.tau = sls.tau;
  d.a2h = sls.alpha2_history;
}

// ---- matrix-free operators: gpss.cpp:117-219 on the host, every reduction, projection,
// steplength rule and backtracking step on the device primitives
GpIterationState generic_gp_init(const Objective& prob, const L1Ball& ball, Vector x0,
                                 const GpConfig& cfg, MatvecCounter& mv) {
  if (x0.size() == 0) x0 = Vector::Zero(prob.dim());
  if (!ball.contains(x0, 1e-12)) throw std::invalid_argument("gp_init: starting point is infeasible");
  GpIterationState st;
  st.x = std::move(x0);
  st.kx_minus_y = prob.op().apply(st.x, mv) - prob.y();
  st.f = st.kx_minus_y.squaredNorm();
  st.grad = 2.0 * prob.op().apply_adjoint(st.kx_minus_y, mv);
  st.alpha0 = alpha0_from_gradient(ball, st.x, st.grad, cfg);
  st.f_history.assign(1, st.f);
  return st;
}

GpStepInfo generic_gp_iterate(const Objective& prob, const L1Ball& ball, const GpConfig& cfg,
                              GpIterationState& st, SteplengthState& sls, MatvecCounter& mv,
                              double tol) {
  GpStepInfo info;
  if (st.stationary) {
    info.stationary = true;
    info.stationarity = 0.0;
    return info;
  }
  if (st.k == 0) info.steplength.alpha = st.alpha0;
  else info.steplength = steplength_select(sls, st.x - sls.prev_x, st.grad - sls.prev_grad, cfg, st.k);
  const double first_alpha = info.steplength.alpha;
  double alpha = first_alpha, first_stat = 0.0;
  Vector d;
  for (bool first = true;; first = false) {  // escalation, gpss.cpp:162-191
    d = project_l1_ball(st.x - alpha * st.grad, ball) - st.x;
    info.stationarity = d.lpNorm<Infinity>();
    if (first) first_stat = info.stationarity;
    if (info.stationarity <= tol) {
      st.stationary = info.stationary = true;
      info.alpha = alpha;
      info.f_after = st.f;
      return info;
    }
    info.dir_derivative = st.grad.dot(d);
    if (info.dir_derivative < 0.0) break;
    if (alpha >= cfg.alpha_max) {
      st.stationary = info.stationary = true;
      info.alpha = first_alpha;
      info.stationarity = first_stat;
      info.f_after = st.f;
      return info;
    }
    alpha = std::min(alpha * 10.0, cfg.alpha_max);
  }
  info.alpha = alpha;
  const Vector kd = prob.op().apply(d, mv);
  info.f_max = *std::max_element(st.f_history.begin(), st.f_history.end());
  const l1g_gp_config c = conv(cfg);
  int32_t h = 0;
  double f_new = 0.0;
  check(l1g_backtrack(ctx(), st.f, st.kx_minus_y.dot(kd), kd.squaredNorm(), info.f_max,
                      info.dir_derivative, &c, &info.step, &f_new, &h));
  info.halvings = h;
  sls.prev_x = st.x;
  sls.prev_grad = st.grad;
  st.x += info.step * d;
  st.kx_minus_y += info.step * kd;
  st.f = f_new;
  st.grad = 2.0 * prob.op().apply_adjoint(st.kx_minus_y, mv);
  st.f_history.push_back(st.f);
  while (st.f_history.size() > static_cast<std::size_t>(cfg.memory)) st.f_history.pop_front();
  ++st.k;
  info.f_after = st.f;
  return info;
}
}  // namespace

// gpss.cpp:117-134
GpIterationState gp_init(const Objective& prob, const L1Ball& ball, Vector x0,
                         const GpConfig& cfg, MatvecCounter& mv) {
  cfg.validate();
  if (x0.size() != 0 && x0.size() != prob.dim())
    throw std::invalid_argument("gp_init: starting point has wrong dimension");
  auto* op = dynamic_cast<const DenseOperator*>(&prob.op());
  if (!op) return generic_gp_init(prob, ball, std::move(x0), cfg, mv);
  auto dev = std::make_shared<DeviceIterationState>();
  dev->n = op->rows();
  dev->p = op->cols();
  dev->cfg = cfg;
  dev->rho = ball.radius();
  const l1g_gp_config c = conv(cfg);
  check(l1g_solver_create(op->handle(), prob.y().data(), ball.radius(), &c, &dev->s));
  check(l1g_solver_init(dev->s, x0.size() ? x0.data() : nullptr));
  mv.count += 2;
  GpIterationState st;
  pull(*dev, st, nullptr);
  st.device = std::move(dev);
  return st;
}

// gpss.cpp:136-219
GpStepInfo gp_iterate(const Objective& prob, const L1Ball& ball, const GpConfig& cfg,
                      GpIterationState& state, SteplengthState& sls, MatvecCounter& mv,
                      double stationarity_tol) {
  if (!state.device) return generic_gp_iterate(prob, ball, cfg, state, sls, mv, stationarity_tol);
  DeviceIterationState& d = *state.device;
  push(d, state, sls, cfg, ball);
  GpStepInfo info;
  if (state.stationary) {  // gpss.cpp:139-143
    info.stationary = true;
    info.stationarity = 0.0;
    return info;
  }
  const int64_t before = solver_matvecs(d.s);
  l1g_iter_record rec;
  int32_t stat = 0;
  check(l1g_solver_iterate(d.s, stationarity_tol, &rec, &stat));
  mv.count += solver_matvecs(d.s) - before;
  const l1g_gp_state g = pull(d, state, &sls);
  info.steplength = conv(g.choice);  // the choice before any escalation (gpss.cpp:148-153)
  info.stationary = stat != 0;
  info.alpha = rec.alpha;
  info.stationarity = rec.stationarity;
  info.f_after = state.f;
  if (!info.stationary) {
    info.step = rec.step;
    info.f_max = rec.f_max;
    info.dir_derivative = rec.dir_derivative;
    info.halvings = rec.halvings;
  } else if (!std::isnan(rec.dir_derivative)) {
    info.dir_derivative = rec.dir_derivative;
  }
  return info;
}

namespace {

// gpss.cpp:221-292 for matrix-free operators: the reference's loop over gp_init / gp_iterate
SolverState generic_solve(const Objective& prob, const L1Ball& ball, const GpConfig& cfg,
                          const StopRule& stop, const IterationCallback& cb, Vector x0) {
  using Clock = std::chrono::steady_clock;
  const auto start = Clock::now();
  auto since = [&] { return std::chrono::duration<double>(Clock::now() - start).count(); };
  SolverState out;
  GpIterationState st = gp_init(prob, ball, std::move(x0), cfg, out.matvecs);
  SteplengthState sls = steplength_init(cfg);
  out.reason = StopReason::MaxIterations;
  out.objective = st.f;
  double f_prev = st.f;
  for (long k = 0;; ++k) {
    if (stop.max_iterations > 0 && k >= stop.max_iterations) {
      out.reason = StopReason::MaxIterations;
      break;
    }
    if (stop.max_matvecs > 0 && out.matvecs.count >= stop.max_matvecs) {
      out.reason = StopReason::MaxMatvecs;
      break;
    }
    if (stop.max_seconds > 0.0 && since() >= stop.max_seconds) {
      out.reason = StopReason::MaxSeconds;
      break;
    }
    const GpStepInfo info = gp_iterate(prob, ball, cfg, st, sls, out.matvecs, stop.stationarity_tol);
    out.stationarity = info.stationarity;
    if (info.stationary) {
      out.reason = StopReason::Stationary;
      break;
    }
    out.iterations = st.k;
    out.objective = st.f;
    out.elapsed_seconds = since();
    if (cb) {
      IterationRecord rec;
      rec.k = k;
      rec.f = info.f_after;
      rec.stationarity = info.stationarity;
      rec.alpha = info.alpha;
      rec.step = info.step;
      rec.matvecs = out.matvecs.count;
      rec.elapsed_seconds = out.elapsed_seconds;
      rec.bb_active = info.steplength.bb_active;
      rec.bb1_raw = info.steplength.bb1_raw;
      rec.bb2_raw = info.steplength.bb2_raw;
      rec.tau_before = info.steplength.tau_before;
      rec.tau_after = info.steplength.tau_after;
      rec.f_max = info.f_max;
      rec.dir_derivative = info.dir_derivative;
      cb(rec, st.x);
    }
    if (stop.objective_tol > 0.0 &&
        std::abs(f_prev - st.f) <= stop.objective_tol * std::max(1.0, std::abs(st.f))) {
      out.reason = StopReason::ObjectiveTol;
      break;
    }
    f_prev = st.f;
  }
  out.x = std::move(st.x);
  out.iterations = st.k;
  out.objective = st.f;
  out.f_history = std::move(st.f_history);
  out.elapsed_seconds = since();
  return out;
}

struct CbCtx {
  const IterationCallback* cb;
  std::exception_ptr err;
};

// a throwing callback stops the device loop at once (nonzero return -> L1G_ECANCELED) and
// its exception is rethrown to the caller, as the reference propagates it
int trampoline(const l1g_iter_record* rec, const double* x, int64_t p, void* user) {
  auto* c = static_cast<CbCtx*>(user);
  if (c->err) return 1;
  try {
    Vector xv(p);
    std::memcpy(xv.data(), x, sizeof(double) * static_cast<std::size_t>(p));
    (*c->cb)(conv(*rec), xv);
    return 0;
  } catch (...) {
    c->err = std::current_exception();
    return 1;
  }
}

}  // namespace

// gpss.cpp:221-292
SolverState gpss_solve(const Objective& prob, const L1Ball& ball, const GpConfig& cfg,
                       const StopRule& stop, const IterationCallback& cb, Vector x0) {
  stop.validate();
  auto* dense = dynamic_cast<const DenseOperator*>(&prob.op());
  if (!dense) return generic_solve(prob, ball, cfg, stop, cb, std::move(x0));
  cfg.validate();
  if (x0.size() != 0 && x0.size() != prob.dim())
    throw std::invalid_argument("gp_init: starting point has wrong dimension");
  const l1g_gp_config c = conv(cfg);
  const l1g_stop_rule s = conv(stop);
  l1g_result res;
  Vector x(prob.dim());
  if (!cb) {
    check(l1g_gpss_solve(dense->handle(), prob.y().data(), ball.radius(), &c, &s,
                         x0.size() ? x0.data() : nullptr, x.data(), &res, nullptr, 0));
    return state_from(res, std::move(x));
  }
  l1g_solver* h = nullptr;
  check(l1g_solver_create(dense->handle(), prob.y().data(), ball.radius(), &c, &h));
  CbCtx cc{&cb, nullptr};
  int rc = l1g_solver_init(h, x0.size() ? x0.data() : nullptr);
  if (rc == L1G_OK) rc = l1g_solver_run_cb(h, &s, &res, &trampoline, &cc);
  if (rc == L1G_OK)
    rc = l1g_solver_get(h, x.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  const std::string msg = rc ? l1g_last_error() : "";
  l1g_solver_destroy(h);
  if (cc.err) std::rethrow_exception(cc.err);
  if (rc == L1G_EINVAL) throw std::invalid_argument(msg);
  if (rc) throw std::runtime_error(msg);
  return state_from(res, std::move(x));
}

namespace {
// psd / ista / fista through the device drivers (l1g_psd_solve, l1g_shrinkage_solve)
SolverState other_solve(const Objective& prob, double param, int kind, const StopRule& stop,
                        const IterationCallback& cb, const char* name) {
  stop.validate();
  auto* dense = dynamic_cast<const DenseOperator*>(&prob.op());
  if (!dense) throw std::invalid_argument(std::string(name) + ": needs a DenseOperator here");
  const l1g_stop_rule s = conv(stop);
  l1g_result res;
  Vector x(prob.dim());
  CbCtx cc{&cb, nullptr};
  const l1g_iter_cb fn = cb ? &trampoline : nullptr;
  const int rc = kind == 0
                     ? l1g_psd_solve(dense->handle(), prob.y().data(), param, &s, x.data(), &res,
                                     nullptr, 0, fn, &cc)
                     : l1g_shrinkage_solve(dense->handle(), prob.y().data(), param, kind == 2, &s,
                                           x.data(), &res, nullptr, 0, fn, &cc);
  if (cc.err) std::rethrow_exception(cc.err);
  if (rc) {
    const std::string msg = l1g_last_error();
    if (rc == L1G_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  return state_from(res, std::move(x));
}
}  // namespace

void save_problem(const GeneratedProblem& prob, const std::filesystem::path& path) {
  if (!prob.op) throw std::invalid_argument("save_problem: problem has no operator");
  if (prob.y.size() != prob.op->rows() || prob.x_true.size() != prob.op->cols())
    throw std::invalid_argument("save_problem: inconsistent problem dimensions");
  check(l1g_problem_save(path.string().c_str(), prob.op->handle(), prob.y.data(),
                         prob.x_true.data(), prob.seed, prob.noise_level));
}

GeneratedProblem load_problem(const std::filesystem::path& path) {
  int64_t n = 0, p = 0;
  check(l1g_problem_info(path.string().c_str(), &n, &p, nullptr, nullptr));
  GeneratedProblem g;
  g.y = Vector(n);
  g.x_true = Vector(p);
  l1g_op* op = nullptr;
  check(l1g_problem_load(ctx(), path.string().c_str(), g.y.data(), g.x_true.data(), &g.seed,
                         &g.noise_level, &op));
  g.op = std::make_shared<DenseOperator>(op, n, p);
  return g;
}

std::uint64_t problem_hash(const GeneratedProblem& prob) {
  std::uint64_t h = 0;
  check(l1g_problem_hash(prob.op->handle(), prob.y.data(), prob.x_true.data(), prob.seed,
                         prob.noise_level, &h));
  return h;
}

SolverState psd_solve(const Objective& prob, const L1Ball& ball, const StopRule& stop,
                      const IterationCallback& cb) {
  return other_solve(prob, ball.radius(), 0, stop, cb, "psd_solve");
}

SolverState ista_solve(const Objective& prob, const PenaltyWeight& lambda, const StopRule& stop,
                       const IterationCallback& cb) {
  return other_solve(prob, lambda.value(), 1, stop, cb, "ista_solve");
}

SolverState fista_solve(const Objective& prob, const PenaltyWeight& lambda, const StopRule& stop,
                        const IterationCallback& cb) {
  return other_solve(prob, lambda.value(), 2, stop, cb, "fista_solve");
}

}  // namespace l1solve

// ------------------------------------------------------------------------- rng, generators
// The reference's small seeded problems (generators.cpp:13-147) for callers and tests:
// std::mt19937_64 uniforms, Box-Muller normals with libm, host arithmetic.
namespace l1solve {

double Rng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1 = uniform();
  while (u1 == 0.0) u1 = uniform();
  const double u2 = uniform();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * M_PI * u2;
  spare_ = radius * std::sin(angle);
  has_spare_ = true;
  return radius * std::cos(angle);
}

std::uint64_t Rng::below(std::uint64_t bound) {
  if (bound == 0) throw std::invalid_argument("Rng::below: bound must be positive");
  const std::uint64_t threshold = (0 - bound) % bound;  // 2^64 mod bound
  for (;;) {
    const std::uint64_t r = engine_();
    if (r >= threshold) return r % bound;
  }
}

Vector Rng::normal_vector(Index n) {
  Vector v(n);
  for (Index i = 0; i < n; ++i) v[i] = normal();
  return v;
}

Matrix Rng::normal_matrix(Index rows, Index cols) {
  Matrix m(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) m(i, j) = normal();
  return m;
}

std::vector<Index> Rng::sample_indices(Index population, Index k) {
  if (k > population) throw std::invalid_argument("Rng::sample_indices: k > population");
  std::vector<Index> pool(static_cast<std::size_t>(population));
  for (Index i = 0; i < population; ++i) pool[static_cast<std::size_t>(i)] = i;
  for (Index i = 0; i < k; ++i) {
    const Index j = i + static_cast<Index>(below(static_cast<std::uint64_t>(population - i)));
    std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(j)]);
  }
  pool.resize(static_cast<std::size_t>(k));
  return pool;
}

namespace {

void check_gen(Index n, Index p, Index nnz, double noise_level) {
  if (n < 1 || p < 1) throw std::invalid_argument("problem generator: n and p must be positive");
  if (nnz < 0 || nnz > p)
    throw std::invalid_argument("problem generator: nnz must lie in [0, p], got " +
                                std::to_string(nnz) + " with p = " + std::to_string(p));
  if (noise_level < 0.0) throw std::invalid_argument("problem generator: noise_level must be >= 0");
}

// spikes of +-1 on a random support, y = K x + e with ||e|| = noise * ||K x||
GeneratedProblem finish_problem(Rng& rng, Matrix k, Index nnz, double noise_level,
                                std::uint64_t seed) {
  GeneratedProblem prob;
  prob.op = std::make_shared<DenseOperator>(k);
  const Index p = k.cols();
  prob.x_true = Vector::Zero(p);
  for (const Index i : rng.sample_indices(p, nnz)) prob.x_true[i] = rng.sign();
  MatvecCounter scratch;
  prob.y = prob.op->apply(prob.x_true, scratch);
  if (noise_level != 0.0) {
    const Vector e = rng.normal_vector(k.rows());
    const double e_norm = e.norm();
    if (e_norm != 0.0) {
      const double signal = prob.y.norm();
      const double scale = (signal > 0.0 ? noise_level * signal : noise_level) / e_norm;
      prob.y += scale * e;
    }
  }
  prob.noise_level = noise_level;
  prob.seed = seed;
  return prob;
}

// thin Q (rows x cols, cols <= rows) of a Householder QR, column by column
Matrix householder_q(Matrix a) {
  const Index m = a.rows(), n = a.cols();
  std::vector<Vector> vs;
  for (Index j = 0; j < n; ++j) {
    double norm = 0.0;
    for (Index i = j; i < m; ++i) norm += a(i, j) * a(i, j);
    norm = std::sqrt(norm);
    Vector v(m);
    const double alpha = a(j, j) > 0.0 ? -norm : norm;
    for (Index i = j; i < m; ++i) v[i] = a(i, j);
    v[j] = v[j] - alpha;
    double vn = 0.0;
    for (Index i = j; i < m; ++i) vn += v[i] * v[i];
    if (vn > 0.0)
      for (Index c = j; c < n; ++c) {
        double dotv = 0.0;
        for (Index i = j; i < m; ++i) dotv += v[i] * a(i, c);
        const double f = 2.0 * dotv / vn;
        for (Index i = j; i < m; ++i) a(i, c) = a(i, c) - f * v[i];
      }
    vs.push_back(std::move(v));
  }
  Matrix q = Matrix::Identity(m, n);
  for (Index j = n - 1; j >= 0; --j) {
    const Vector& v = vs[static_cast<std::size_t>(j)];
    double vn = 0.0;
    for (Index i = j; i < m; ++i) vn += v[i] * v[i];
    if (vn == 0.0) continue;
    for (Index c = 0; c < n; ++c) {
      double dotv = 0.0;
      for (Index i = j; i < m; ++i) dotv += v[i] * q(i, c);
      const double f = 2.0 * dotv / vn;
      for (Index i = j; i < m; ++i) q(i, c) = q(i, c) - f * v[i];
    }
  }
  return q;
}

}  // namespace

// generators.cpp:99-117
GeneratedProblem gen_gaussian_problem(Index n, Index p, Index nnz, double noise_level,
                                      std::uint64_t seed) {
  check_gen(n, p, nnz, noise_level);
  Rng rng(seed);
  Matrix k = rng.normal_matrix(n, p);
  {
    const DenseOperator raw(k);
    const double sigma = spectral_norm_estimate(raw, 1000, 1e-8);
    if (sigma == 0.0) throw std::runtime_error("gen_gaussian_problem: degenerate matrix");
    k /= sigma;
  }
  return finish_problem(rng, std::move(k), nnz, noise_level, seed);
}

// generators.cpp:119-147: singular values decay^(i-1) between Gaussian orthonormal factors
GeneratedProblem gen_illconditioned_problem(Index n, Index p, Index nnz, double decay,
                                            double noise_level, std::uint64_t seed) {
  check_gen(n, p, nnz, noise_level);
  if (!(decay > 0.0 && decay < 1.0))
    throw std::invalid_argument("gen_illconditioned_problem: decay must lie strictly in (0,1)");
  Rng rng(seed);
  const Index r = std::min(n, p);
  const Matrix u = householder_q(rng.normal_matrix(n, r));
  const Matrix v = householder_q(rng.normal_matrix(p, r));
  Matrix k(n, p);
  double s = 1.0;
  for (Index l = 0; l < r; ++l, s *= decay)
    for (Index j = 0; j < p; ++j)
      for (Index i = 0; i < n; ++i) k(i, j) = k(i, j) + u(i, l) * (s * v(j, l));
  return finish_problem(rng, std::move(k), nnz, noise_level, seed);
}

// ------------------------------------------------------------------------- reference minimizer
// reference.cpp:9-13
double penalized_fixed_point_residual(const Objective& prob, const Vector& x, double lambda,
                                      MatvecCounter& mv) {
  const Vector r = prob.residual(x, mv);
  return (x - soft_threshold(x + r, lambda)).lpNorm<Infinity>();
}

// reference.cpp:38-82 (DenseOperator: the device driver l1g_reference_minimizer)
ReferenceSolution reference_minimizer(const Objective& prob, double lambda,
                                      const ReferenceOptions& opt) {
  if (!(lambda > 0.0)) throw std::invalid_argument("reference_minimizer: lambda must be > 0");
  auto* dense = dynamic_cast<const DenseOperator*>(&prob.op());
  ReferenceSolution ref;
  ref.lambda = lambda;
  ref.oracle_tol = opt.oracle_tol;
  if (dense) {
    l1g_ref_options o{opt.oracle_tol, opt.max_iterations, opt.check_interval, opt.nnz_threshold};
    l1g_ref_solution out;
    ref.x = Vector(prob.dim());
    check(l1g_reference_minimizer(dense->handle(), prob.y().data(), lambda, &o, ref.x.data(),
                                  &out));
    ref.rho = out.rho;
    ref.nnz = static_cast<long>(out.nnz);
    ref.certificate = out.certificate;
    return ref;
  }
  // matrix-free operator: the reference's loop over the device primitives
  MatvecCounter mv;
  const double lmax = lambda_max(prob.op(), prob.y(), mv);
  Vector x = Vector::Zero(prob.dim());
  double cert = 0.0;
  bool ok = lambda >= lmax;
  if (ok) {
    cert = penalized_fixed_point_residual(prob, x, lambda, mv);
  } else {
    const double c2 = kShrinkageOperatorScale * kShrinkageOperatorScale;
    const double lam_eff = lambda * c2;
    Vector x_prev = x;
    double t = 1.0;
    for (long k = 0; k < opt.max_iterations && !ok; ++k) {
      const double t_next = fista_t_next(t);
      const Vector point = x + ((t - 1.0) / t_next) * (x - x_prev);
      const Vector misfit = prob.op().apply(point, mv) - prob.y();
      const Vector grad_half = prob.op().apply_adjoint(misfit, mv);
      Vector x_new = soft_threshold(point - c2 * grad_half, lam_eff);
      x_prev = std::move(x);
      x = std::move(x_new);
      t = t_next;
      const double surrogate = (x - point).lpNorm<Infinity>();
      if ((k + 1) % opt.check_interval == 0 || surrogate <= opt.oracle_tol) {
        cert = penalized_fixed_point_residual(prob, x, lambda, mv);
        ok = cert <= opt.oracle_tol;
      }
    }
    if (!ok) {
      MatvecCounter scratch;
      cert = penalized_fixed_point_residual(prob, x, lambda, scratch);
      throw std::runtime_error("reference_minimizer: certificate " + std::to_string(cert) +
                               " did not reach tolerance " + std::to_string(opt.oracle_tol) +
                               " within " + std::to_string(opt.max_iterations) +
                               " iterations (lambda = " + std::to_string(lambda) + ")");
    }
  }
  ref.rho = x.lpNorm<1>();
  for (Index i = 0; i < x.size(); ++i) ref.nnz += std::abs(x[i]) > opt.nnz_threshold;
  ref.certificate = cert;
  ref.x = std::move(x);
  return ref;
}

}  // namespace l1solve
