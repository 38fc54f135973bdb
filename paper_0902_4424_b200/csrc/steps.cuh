// steps.cuh -- the scalar tails of gp_iterate run by the finish kernels (one thread), shared
// by the single-RHS finishes (gemv.cu) and the batched ones (dmma.cu).
#pragma once
#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"

namespace l1g {

// warp-cooperative copy of the device state into shared memory (one coalesced pass)
__device__ __forceinline__ void snapshot(DevState* dst, const DevState* src, int lane) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
  for (int i = lane; i < (int)(sizeof(DevState) / 8); i += 32) d[i] = __ldcg(s + i);
  __syncwarp();
}

// a run leaves RUNNING: batched runs count their live problems down
__device__ __forceinline__ void leave_run(DevState* st, int status) {
  st->status = status;
  if (st->nrun) atomicSub(st->nrun, 1);
}

// after K x0 (FWD_INIT: f = ||K x0 - y||^2, gpss.cpp:128-133) or K d (FWD_ITER: a = r'Kd,
// b = ||Kd||^2, nonmonotone reference and quadratic backtracking, gpss.cpp:195-203)
__device__ __forceinline__ void fwd_tail(DevState* st, const DevState& s, int mode, double A,
                                         double B) {
  if (mode == FWD_INIT) {
    st->f = A;
    st->f_prev = A;
    st->fh[0] = A;
    st->fh_len = 1;
    return;
  }
  st->a = A;
  st->b = B;
  double f_max = s.fh[0];
  for (int i = 1; i < s.fh_len; ++i) f_max = s.fh[i] > f_max ? s.fh[i] : f_max;
  st->f_max = f_max;
  double step, f_new;
  int h;
  if (backtrack_quadratic(s.f, A, B, f_max, s.gd, s.cfg, &step, &f_new, &h)) {
    st->step = step;
    st->f_new = f_new;
    st->halvings = h;
  } else {
    st->failure = FAIL_BACKTRACK;
    leave_run(st, FAILED);
  }
}

// after g' = 2 K^T r': gpss.cpp:206-217 state advance, gpss.cpp:255-283 loop bookkeeping
// (on the snapshot s, then written back field by field)
__device__ __forceinline__ void adj_tail(DevState* st, DevState& s, double SZ, double SS,
                                         double ZZ) {
  st->sz = SZ;
  st->ss = SS;
  st->zz = ZZ;
  const double f = s.f_new;
  st->f = f;
  int fl = s.fh_len;
  if (fl < kMaxHist) {
    s.fh[fl++] = f;
  } else {
    for (int i = 0; i + 1 < fl; ++i) s.fh[i] = s.fh[i + 1];
    s.fh[fl - 1] = f;
  }
  while (fl > s.cfg.memory) {
    for (int i = 0; i + 1 < fl; ++i) s.fh[i] = s.fh[i + 1];
    --fl;
  }
  for (int i = 0; i < fl; ++i) st->fh[i] = s.fh[i];
  st->fh_len = fl;
  const int64_t k = s.k;
  st->k = k + 1;
  const int64_t mv = s.matvecs + 2;
  st->matvecs = mv;
  l1g_iter_record rec;
  rec.k = k;
  rec.f = f;
  rec.stationarity = s.stat;
  rec.alpha = s.alpha_used;
  rec.step = s.step;
  rec.matvecs = mv;
  rec.elapsed_seconds = elapsed_s(&s);
  rec.bb_active = s.choice.bb_active;
  rec.halvings = s.halvings;
  rec.bb1_raw = s.choice.bb1_raw;
  rec.bb2_raw = s.choice.bb2_raw;
  rec.tau_before = s.choice.tau_before;
  rec.tau_after = s.choice.tau_after;
  rec.f_max = s.f_max;
  rec.dir_derivative = s.gd;
  rec.theta = s.theta;
  rec.support = s.support;
  st->last = rec;
  if (s.trace && k < s.trace_cap) s.trace[k] = rec;
  if (!s.single_step && s.objective_tol > 0.0) {
    const double af = fabs(f);
    if (fabs(sub(s.f_prev, f)) <= mul(s.objective_tol, af > 1.0 ? af : 1.0)) {
      st->reason = L1G_OBJECTIVE_TOL;
      leave_run(st, STOPPED);
    }
  }
  st->f_prev = f;
  st->cur = s.cur ^ 1;
}

}  // namespace l1g
