// scalar.cuh -- the scalar control logic of gpss.cpp, executed by one device thread.
#pragma once
#include "common.cuh"
#include "engine.h"

namespace l1g {

// gpss.cpp:18-20
__host__ __device__ __forceinline__ double clamp_step(double a, const l1g_gp_config& c) {
  const double lo = a < c.alpha_max ? a : c.alpha_max;
  return c.alpha_min > lo ? c.alpha_min : lo;
}

// gpss.cpp:25-37 -- first lambda in {1, theta, theta^2, ...} with
// f0 + 2 a lambda + b lambda^2 <= f_max + beta lambda gd; returns false after 60 shrinks.
__device__ __forceinline__ bool backtrack_quadratic(double f0, double a, double b, double f_max,
                                                    double gd, const l1g_gp_config& c,
                                                    double* step, double* f_new, int* halvings) {
  double lam = 1.0;
  for (int h = 0; h <= 60; ++h) {
    // ((f0 + (2*a)*lam) + (b*lam)*lam) <= f_max + (beta*lam)*gd, each op rounded
    const double f_trial = add(add(f0, mul(mul(2.0, a), lam)), mul(mul(b, lam), lam));
    if (f_trial <= add(f_max, mul(mul(c.beta, lam), gd))) {
      *step = lam;
      *f_new = f_trial;
      *halvings = h;
      return true;
    }
    lam = mul(lam, c.theta);
  }
  return false;
}

// gpss.cpp:59-91 evaluated on the secant dots sz = s'z, ss = s's, zz = z'z
__device__ __forceinline__ void steplength_from_dots(double* tau, double* hist, int* hist_len,
                                                     double sz, double ss, double zz,
                                                     const l1g_gp_config& c, l1g_sl_choice* o) {
  o->tau_before = *tau;
  o->tau_after = *tau;
  o->bb_active = 0;
  o->bb1_raw = __longlong_as_double(0x7ff8000000000000ll);
  o->bb2_raw = __longlong_as_double(0x7ff8000000000000ll);
  if (sz <= 0.0) {
    o->alpha = c.alpha_max;
    return;
  }
  o->bb_active = 1;
  o->bb1_raw = dvd(ss, sz);
  o->bb2_raw = dvd(sz, zz);
  const double a1 = clamp_step(o->bb1_raw, c);
  const double a2 = clamp_step(o->bb2_raw, c);
  hist[(*hist_len)++] = a2;
  while (*hist_len > c.alpha2_memory + 1) {
    for (int i = 0; i + 1 < *hist_len; ++i) hist[i] = hist[i + 1];
    --*hist_len;
  }
  if (dvd(a2, a1) <= *tau) {
    double mn = hist[0];
    for (int i = 1; i < *hist_len; ++i) mn = hist[i] < mn ? hist[i] : mn;
    o->alpha = mn;
    *tau = mul(*tau, 0.9);
  } else {
    o->alpha = a1;
    *tau = mul(*tau, 1.1);
  }
  o->tau_after = *tau;
}

__device__ __forceinline__ double nan_d() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ __forceinline__ double elapsed_s(const DevState* st) {
  return (double)(globaltimer() - st->t_start) * 1e-9;
}

}  // namespace l1g
