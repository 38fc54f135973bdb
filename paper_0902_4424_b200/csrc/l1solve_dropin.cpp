// l1solve_dropin.cpp -- the reference's C++ solver API (include/l1solve/*.hpp) on top of
// the C-ABI (include/l1g.h).  Builds into libl1solve_b200.so, linked against libl1g.so.
//
// DenseOperator problems run the device-resident loop (l1g_gpss_solve / l1g_solver_*).
// A user-defined LinearOperator (matrix-free K) keeps the reference's host-driven loop
// (gpss.cpp:117-292 restated below) with every reduction, the projection, the steplength
// rule and the backtracking executed by the same device code.
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "l1g.h"
#include "l1solve/gpss.hpp"
#include "l1solve/problem_io.hpp"

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
GpIterationState::GpIterationState() = default;
GpIterationState::~GpIterationState() { l1g_solver_destroy(s_); }
GpIterationState::GpIterationState(GpIterationState&& o) noexcept
    : stationary(o.stationary), s_(o.s_) {
  o.s_ = nullptr;
}
GpIterationState& GpIterationState::operator=(GpIterationState&& o) noexcept {
  if (this != &o) {
    l1g_solver_destroy(s_);
    s_ = o.s_;
    stationary = o.stationary;
    o.s_ = nullptr;
  }
  return *this;
}

Vector GpIterationState::x() const {
  Vector v(p_);
  check(l1g_solver_get(s_, v.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
  return v;
}
Vector GpIterationState::kx_minus_y() const {
  Vector v(n_);
  check(l1g_solver_get(s_, nullptr, v.data(), nullptr, nullptr, nullptr, nullptr, nullptr));
  return v;
}
Vector GpIterationState::grad() const {
  Vector v(p_);
  check(l1g_solver_get(s_, nullptr, nullptr, v.data(), nullptr, nullptr, nullptr, nullptr));
  return v;
}
double GpIterationState::f() const {
  double f = 0.0;
  check(l1g_solver_get(s_, nullptr, nullptr, nullptr, &f, nullptr, nullptr, nullptr));
  return f;
}
long GpIterationState::k() const {
  int64_t k = 0;
  check(l1g_solver_get(s_, nullptr, nullptr, nullptr, nullptr, &k, nullptr, nullptr));
  return static_cast<long>(k);
}
double GpIterationState::alpha0() const {
  double a = 0.0;
  check(l1g_solver_get(s_, nullptr, nullptr, nullptr, nullptr, nullptr, &a, nullptr));
  return a;
}

namespace {
const DenseOperator& dense_or_throw(const Objective& prob) {
  auto* d = dynamic_cast<const DenseOperator*>(&prob.op());
  if (!d) throw std::invalid_argument("gp_init/gp_iterate: the device state needs a DenseOperator");
  return *d;
}
int64_t solver_matvecs(l1g_solver* s) {
  int64_t mv = 0;
  check(l1g_solver_get(s, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &mv));
  return mv;
}
}  // namespace

// gpss.cpp:117-134
GpIterationState gp_init(const Objective& prob, const L1Ball& ball, Vector x0,
                         const GpConfig& cfg, MatvecCounter& mv) {
  cfg.validate();
  const DenseOperator& op = dense_or_throw(prob);
  if (x0.size() != 0 && x0.size() != prob.dim())
    throw std::invalid_argument("gp_init: starting point has wrong dimension");
  GpIterationState st;
  st.n_ = op.rows();
  st.p_ = op.cols();
  const l1g_gp_config c = conv(cfg);
  check(l1g_solver_create(op.handle(), prob.y().data(), ball.radius(), &c, &st.s_));
  check(l1g_solver_init(st.s_, x0.size() ? x0.data() : nullptr));
  mv.count += 2;
  return st;
}

// gpss.cpp:136-219
GpStepInfo gp_iterate(const Objective& prob, const L1Ball& ball, const GpConfig& cfg,
                      GpIterationState& state, SteplengthState& sls, MatvecCounter& mv,
                      double stationarity_tol) {
  (void)prob;
  (void)ball;
  (void)cfg;
  (void)sls;
  const int64_t before = solver_matvecs(state.handle());
  l1g_iter_record rec;
  int32_t stat = 0;
  check(l1g_solver_iterate(state.handle(), stationarity_tol, &rec, &stat));
  mv.count += solver_matvecs(state.handle()) - before;
  state.stationary = stat != 0;
  GpStepInfo info;
  info.stationary = stat != 0;
  info.alpha = rec.alpha;
  info.step = rec.step;
  info.f_after = rec.f;
  info.stationarity = rec.stationarity;
  info.f_max = rec.f_max;
  info.dir_derivative = rec.dir_derivative;
  info.halvings = rec.halvings;
  info.steplength.alpha = rec.alpha;
  info.steplength.bb_active = rec.bb_active != 0;
  info.steplength.bb1_raw = rec.bb1_raw;
  info.steplength.bb2_raw = rec.bb2_raw;
  info.steplength.tau_before = rec.tau_before;
  info.steplength.tau_after = rec.tau_after;
  return info;
}

namespace {

// Host-driven loop for matrix-free operators: gpss.cpp:117-292 restated over the device
// primitives (projection, reductions, steplength rule, backtracking).
SolverState generic_solve(const Objective& prob, const L1Ball& ball, const GpConfig& cfg,
                          const StopRule& stop, const IterationCallback& cb, Vector x0) {
  using Clock = std::chrono::steady_clock;
  const auto start = Clock::now();
  auto since = [&] { return std::chrono::duration<double>(Clock::now() - start).count(); };
  SolverState out;
  cfg.validate();
  if (x0.size() == 0) x0 = Vector::Zero(prob.dim());
  if (x0.size() != prob.dim()) throw std::invalid_argument("gp_init: starting point has wrong dimension");
  if (!ball.contains(x0, 1e-12)) throw std::invalid_argument("gp_init: starting point is infeasible");
  Vector x = std::move(x0);
  Vector r = prob.op().apply(x, out.matvecs) - prob.y();
  double f = r.squaredNorm();
  Vector g = 2.0 * prob.op().apply_adjoint(r, out.matvecs);
  const double alpha0 = alpha0_from_gradient(ball, x, g, cfg);
  std::deque<double> fh(1, f);
  SteplengthState sls = steplength_init(cfg);
  Vector xp, gp;
  out.reason = StopReason::MaxIterations;
  out.objective = f;
  double f_prev = f;
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
    SteplengthChoice ch;
    if (k == 0) ch.alpha = alpha0;
    else ch = steplength_select(sls, x - xp, g - gp, cfg, k);
    const double first_alpha = ch.alpha;
    double alpha = first_alpha, first_stat = 0.0, stat = 0.0, gd = 0.0;
    Vector d;
    bool stationary = false;
    for (bool first = true;; first = false) {
      const Vector h = project_l1_ball(x - alpha * g, ball);
      d = h - x;
      stat = d.lpNorm<Infinity>();
      if (first) first_stat = stat;
      if (stat <= stop.stationarity_tol) {
        stationary = true;
        break;
      }
      gd = g.dot(d);
      if (gd < 0.0) break;
      if (alpha >= cfg.alpha_max) {
        stationary = true;
        stat = first_stat;
        break;
      }
      alpha = std::min(alpha * 10.0, cfg.alpha_max);
    }
    out.stationarity = stat;
    if (stationary) {
      out.reason = StopReason::Stationary;
      break;
    }
    const Vector kd = prob.op().apply(d, out.matvecs);
    double f_max = fh.front();
    for (double v : fh) f_max = v > f_max ? v : f_max;
    const l1g_gp_config c = conv(cfg);
    double step = 0.0, f_new = 0.0;
    int32_t halv = 0;
    check(l1g_backtrack(ctx(), f, r.dot(kd), kd.squaredNorm(), f_max, gd, &c, &step, &f_new,
                        &halv));
    xp = x;
    gp = g;
    x += step * d;
    r += step * kd;
    f = f_new;
    g = 2.0 * prob.op().apply_adjoint(r, out.matvecs);
    fh.push_back(f);
    while (fh.size() > static_cast<std::size_t>(cfg.memory)) fh.pop_front();
    out.iterations = k + 1;
    out.objective = f;
    out.elapsed_seconds = since();
    if (cb) {
      IterationRecord rec;
      rec.k = k;
      rec.f = f;
      rec.stationarity = stat;
      rec.alpha = alpha;
      rec.step = step;
      rec.matvecs = out.matvecs.count;
      rec.elapsed_seconds = out.elapsed_seconds;
      rec.bb_active = ch.bb_active;
      rec.bb1_raw = ch.bb1_raw;
      rec.bb2_raw = ch.bb2_raw;
      rec.tau_before = ch.tau_before;
      rec.tau_after = ch.tau_after;
      rec.f_max = f_max;
      rec.dir_derivative = gd;
      cb(rec, x);
    }
    if (stop.objective_tol > 0.0 &&
        std::abs(f_prev - f) <= stop.objective_tol * std::max(1.0, std::abs(f))) {
      out.reason = StopReason::ObjectiveTol;
      break;
    }
    f_prev = f;
  }
  out.x = std::move(x);
  out.f_history = std::move(fh);
  out.elapsed_seconds = since();
  return out;
}

struct CbCtx {
  const IterationCallback* cb;
  std::exception_ptr err;
};

void trampoline(const l1g_iter_record* rec, const double* x, int64_t p, void* user) {
  auto* c = static_cast<CbCtx*>(user);
  if (c->err) return;
  try {
    Vector xv(p);
    std::memcpy(xv.data(), x, sizeof(double) * static_cast<std::size_t>(p));
    (*c->cb)(conv(*rec), xv);
  } catch (...) {
    c->err = std::current_exception();
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
