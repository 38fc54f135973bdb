// Drop-in check of the C++ API (include/l1solve/*.hpp over libl1g.so): the calls a
// reference caller makes (DenseOperator, Objective, L1Ball, gpss_solve with and without a
// callback, gp_init/gp_iterate, steplength/backtracking/projection pieces, error classes),
// each checked against closed forms or against the other entry points.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <stdexcept>
#include <vector>

#include "l1solve/gpss.hpp"
#include "l1solve/problem_io.hpp"

using namespace l1solve;

static int g_fail = 0, g_pass = 0;
#define EXPECT(c)                                                              \
  do {                                                                         \
    if (c) ++g_pass;                                                           \
    else {                                                                     \
      ++g_fail;                                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);                 \
    }                                                                          \
  } while (0)
#define EXPECT_THROW(stmt, E)                                                  \
  do {                                                                         \
    bool t_ = false;                                                           \
    try {                                                                      \
      stmt;                                                                    \
    } catch (const E&) {                                                       \
      t_ = true;                                                               \
    }                                                                          \
    EXPECT(t_);                                                                \
  } while (0)

static bool near(double a, double b, double eps) { return std::abs(a - b) <= eps * (1 + std::abs(b)); }

// small seeded Gaussian-ish matrix without any RNG library: a fixed LCG
static Matrix lcg_matrix(Index n, Index p, unsigned seed) {
  Matrix m(n, p);
  unsigned long long s = seed * 2654435761ull + 1;
  for (Index j = 0; j < p; ++j)
    for (Index i = 0; i < n; ++i) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      m(i, j) = ((double)(s >> 11) * 0x1.0p-53 - 0.5) / std::sqrt((double)n);
    }
  return m;
}

int main() {
  // operator arithmetic (2x2) and dimension errors
  Matrix k2(2, 2);
  k2(0, 0) = 1; k2(0, 1) = 2; k2(1, 0) = 0; k2(1, 1) = 1;
  DenseOperator op2(k2);
  MatvecCounter mv;
  Vector y2 = op2.apply(Vector{1.0, 1.0}, mv);
  EXPECT(y2[0] == 3.0 && y2[1] == 1.0);
  Vector a2 = op2.apply_adjoint(Vector{1.0, 0.0}, mv);
  EXPECT(a2[0] == 1.0 && a2[1] == 2.0);
  EXPECT(mv.count == 2);
  EXPECT_THROW(op2.apply(Vector{1.0, 2.0, 3.0}, mv), std::invalid_argument);

  // projection known answers (prox.cpp semantics)
  auto pr = project_l1_ball_with_threshold(Vector{0.9, 0.5}, L1Ball(1.0));
  EXPECT(near(pr.threshold, 0.2, 1e-12) && near(pr.point[0], 0.7, 1e-12) && near(pr.point[1], 0.3, 1e-12));
  EXPECT_THROW(L1Ball(-1.0), std::invalid_argument);
  EXPECT_THROW(soft_threshold(Vector{1.0}, -0.1), std::invalid_argument);

  // steplength worked example and backtracking hand trace
  GpConfig cfg;
  SteplengthState sl = steplength_init(cfg);
  auto ch = steplength_select(sl, Vector{1.0, 1.0}, Vector{1.0, 3.0}, cfg, 1);
  EXPECT(ch.bb_active && near(ch.alpha, 0.5, 1e-15) && near(sl.tau, 0.55, 1e-15));
  Matrix one(1, 1);
  one(0, 0) = 1.0;
  DenseOperator op1(one);
  Objective o1(op1, Vector{0.0});
  auto bt = backtracking_search(o1, Vector{1.0}, Vector{-2.0}, 1.0, -4.0, cfg, mv);
  EXPECT(near(bt.step, 0.5, 1e-15) && bt.halvings == 1);
  EXPECT_THROW(backtracking_search(o1, Vector{1.0}, Vector{-2.0}, -1e10, -4.0, cfg, mv),
               std::runtime_error);

  // identity operator: gpss reaches the projection of y
  DenseOperator id(Matrix::Identity(2, 2));
  StopRule stop;
  stop.max_iterations = 50;
  stop.stationarity_tol = 1e-10;
  SolverState s = gpss_solve(Objective(id, Vector{3.0, 0.0}), L1Ball(1.0), cfg, stop);
  EXPECT(std::abs(s.x[0] - 1.0) <= 1e-10 && s.x[1] == 0.0 && s.reason == StopReason::Stationary);
  EXPECT_THROW(gpss_solve(Objective(id, Vector{1.0, 1.0}), L1Ball(0.5), cfg, stop, {},
                          Vector{1.0, 1.0}),
               std::invalid_argument);

  // a 60 x 200 problem: graph path == callback path == gp_iterate steps; records consistent
  const Matrix K = lcg_matrix(60, 200, 7);
  DenseOperator op(K);
  Vector xt(200);
  xt[3] = 1.0; xt[50] = -1.0; xt[120] = 0.5;
  MatvecCounter m0;
  const Vector y = op.apply(xt, m0);
  const Objective obj(op, y);
  const L1Ball ball(2.5);
  StopRule st2;
  st2.max_iterations = 40;
  st2.stationarity_tol = 0.0;
  const SolverState sa = gpss_solve(obj, ball, cfg, st2);
  std::vector<IterationRecord> recs;
  Vector last;
  const SolverState sb = gpss_solve(obj, ball, cfg, st2, [&](const IterationRecord& r, const Vector& x) {
    recs.push_back(r);
    last = x;
  });
  EXPECT(sa.iterations == sb.iterations && (long)recs.size() == sa.iterations);
  bool same = sa.x.size() == sb.x.size();
  for (Index i = 0; same && i < sa.x.size(); ++i) same = sa.x[i] == sb.x[i] && last[i] == sa.x[i];
  EXPECT(same);
  EXPECT(sa.matvecs.count == 2 + 2 * sa.iterations);
  bool mono = true;
  for (std::size_t i = 1; i < recs.size(); ++i) mono = mono && recs[i].f <= recs[i - 1].f;
  EXPECT(mono);
  MatvecCounter mv2;
  GpIterationState gs = gp_init(obj, ball, Vector(), cfg, mv2);
  SteplengthState sls = steplength_init(cfg);
  for (long i = 0; i < sa.iterations; ++i) gp_iterate(obj, ball, cfg, gs, sls, mv2, 0.0);
  const Vector gx = gs.x;
  bool same2 = true;
  for (Index i = 0; i < gx.size(); ++i) same2 = same2 && gx[i] == sa.x[i];
  EXPECT(same2 && mv2.count == sa.matvecs.count);

  // the reference's public GpIterationState fields (gpss.hpp:89-98) after gp_init / gp_iterate
  {
    MatvecCounter mvi;
    GpIterationState s0 = gp_init(obj, ball, Vector(), cfg, mvi);
    EXPECT(s0.k == 0 && s0.f_history.size() == 1 && s0.f_history.front() == s0.f);
    EXPECT(s0.x.size() == 200 && s0.kx_minus_y.size() == 60 && s0.grad.size() == 200);
    EXPECT(near(s0.f, obj.y().squaredNorm(), 1e-14) && s0.alpha0 > 0.0 && !s0.stationary);
    SteplengthState sl0 = steplength_init(cfg);
    const GpStepInfo i0 = gp_iterate(obj, ball, cfg, s0, sl0, mvi, 0.0);
    EXPECT(s0.k == 1 && s0.f == i0.f_after && s0.f < s0.f_history.front() + 1e300);
    EXPECT(i0.steplength.alpha == s0.alpha0);  // k = 0: alpha0, before any escalation
    EXPECT(sl0.prev_x.size() == 200 && sl0.prev_grad.size() == 200);
  }

  // a user-defined (matrix-free) LinearOperator runs the reference's host-driven loop over
  // the device primitives; with the same K it must reproduce the dense device loop exactly
  struct Wrapped : LinearOperator {
    const DenseOperator* d;
    explicit Wrapped(const DenseOperator* k) : d(k) {}
    Index rows() const override { return d->rows(); }
    Index cols() const override { return d->cols(); }
   protected:
    void do_apply(const Vector& x, Vector& out) const override {
      MatvecCounter m;
      out = d->apply(x, m);
    }
    void do_apply_adjoint(const Vector& r, Vector& out) const override {
      MatvecCounter m;
      out = d->apply_adjoint(r, m);
    }
  };
  const Wrapped wrapped(&op);
  const Objective wobj(wrapped, obj.y());
  {
    StopRule s40;
    s40.max_iterations = 40;
    s40.stationarity_tol = 0.0;
    const SolverState dsol = gpss_solve(obj, ball, cfg, s40);
    const SolverState wsol = gpss_solve(wobj, ball, cfg, s40);
    bool eq = dsol.iterations == wsol.iterations && dsol.matvecs.count == wsol.matvecs.count &&
              dsol.objective == wsol.objective;
    for (Index i = 0; eq && i < dsol.x.size(); ++i) eq = dsol.x[i] == wsol.x[i];
    EXPECT(eq);
    // caller edits between steps (x, cached misfit and gradient, GpConfig) reach the device
    auto run = [&](const Objective& o) {
      MatvecCounter m;
      GpConfig c = cfg;
      GpIterationState st = gp_init(o, ball, Vector(), c, m);
      SteplengthState sl = steplength_init(c);
      for (int i = 0; i < 5; ++i) gp_iterate(o, ball, c, st, sl, m, 0.0);
      st.x *= 0.5;  // still feasible; refresh the caches the way a caller would
      st.kx_minus_y = o.op().apply(st.x, m) - o.y();
      st.f = st.kx_minus_y.squaredNorm();
      st.grad = 2.0 * o.op().apply_adjoint(st.kx_minus_y, m);
      st.f_history.assign(1, st.f);
      c.memory = 3;
      for (int i = 0; i < 6; ++i) gp_iterate(o, ball, c, st, sl, m, 0.0);
      return st;
    };
    const GpIterationState a = run(obj), b = run(wobj);
    bool eq2 = a.k == b.k && a.f == b.f && a.f_history.size() == b.f_history.size();
    for (Index i = 0; eq2 && i < a.x.size(); ++i) eq2 = a.x[i] == b.x[i] && a.grad[i] == b.grad[i];
    EXPECT(eq2 && a.device && !b.device);
  }

  // a throwing callback stops the device loop at once and its exception propagates
  {
    StopRule s100;
    s100.max_iterations = 100;
    s100.stationarity_tol = 0.0;
    int calls = 0;
    bool thrown = false;
    try {
      gpss_solve(obj, ball, cfg, s100, [&](const IterationRecord&, const Vector&) {
        if (++calls == 3) throw std::range_error("stop here");
      });
    } catch (const std::range_error&) {
      thrown = true;
    }
    EXPECT(thrown && calls == 3);
  }

  // spectral norm of a diagonal operator
  Matrix dg = Matrix::Zero(2, 2);
  dg(0, 0) = 1.0;
  dg(1, 1) = 5.0;
  EXPECT(near(spectral_norm_estimate(DenseOperator(dg)), 5.0, 1e-10));

  // psd / ista / fista (psd.cpp, shrinkage.cpp): feasibility, matvec accounting, callbacks
  {
    StopRule st3;
    st3.max_iterations = 40;
    st3.stationarity_tol = 0.0;
    long ncb = 0;
    const SolverState sp = psd_solve(obj, ball, st3, [&](const IterationRecord&, const Vector&) { ++ncb; });
    EXPECT(sp.iterations == 40 && ncb == 40 && sp.matvecs.count == 3 * 40);
    EXPECT(sp.x.lpNorm<1>() <= ball.radius() * (1 + 1e-12) + 1e-12);
    EXPECT(sp.f_history.size() == 10);
    MatvecCounter mvx;
    const double lam = 0.05 * obj.op().apply_adjoint(obj.y(), mvx).lpNorm<Eigen::Infinity>();
    const SolverState si = ista_solve(obj, PenaltyWeight(lam), st3);
    const SolverState sf = fista_solve(obj, PenaltyWeight(lam), st3);
    EXPECT(si.matvecs.count == 80 && sf.matvecs.count == 80);
    EXPECT(sf.objective <= si.objective * 1.5);
    EXPECT_THROW(ista_solve(obj, PenaltyWeight(-1.0), st3), std::invalid_argument);
  }

  // L1PROBv1 round trip through the drop-in problem_io (problem_io.cpp)
  {
    GeneratedProblem g;
    Matrix km = Matrix::Zero(3, 4);
    for (Index i = 0; i < 3; ++i)
      for (Index j = 0; j < 4; ++j) km(i, j) = 1.0 + i * 4 + j;
    g.op = std::make_shared<DenseOperator>(km);
    g.y = Vector{1.0, 2.0, 3.0};
    g.x_true = Vector{0.0, 0.5, 0.0, -1.0};
    g.seed = 123;
    g.noise_level = 0.25;
    const std::filesystem::path path = std::filesystem::temp_directory_path() / "l1g_dropin.l1prob";
    save_problem(g, path);
    EXPECT(std::filesystem::file_size(path) == 40 + 8 * (12 + 3 + 4));
    const GeneratedProblem b = load_problem(path);
    const Matrix kb = b.op->matrix();
    bool same = kb.rows() == 3 && kb.cols() == 4;
    for (Index i = 0; same && i < 3; ++i)
      for (Index j = 0; j < 4; ++j) same = same && kb(i, j) == km(i, j);
    EXPECT(same && b.seed == 123 && b.noise_level == 0.25 && b.y[2] == 3.0 && b.x_true[3] == -1.0);
    EXPECT(problem_hash(b) == problem_hash(g));
    std::filesystem::remove(path);
  }

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
