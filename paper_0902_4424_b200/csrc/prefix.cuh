// prefix.cuh -- exact parallel emulation of a sequential floating-point cumulative sum
// (the sort-and-scan threshold of prox.cpp:43-52), used by project.cu.
#pragma once
#include "common.cuh"

namespace l1g {

#ifndef L1G_PREFIX_PT
#define L1G_PREFIX_PT 512
#endif

// The reference's break test  m > fl((S - rho) / k)  (prox.cpp:47-48) without a division on
// the common path: with a = fl(S - rho), m*k and a are compared with a 2^-50 relative margin
// (both roundings are <= 2^-53); only a near-tie pays for the correctly rounded division.
__device__ __forceinline__ bool passes(double m, double S, double rho, long long k) {
  const double a = sub(S, rho);
  const double kd = (double)k;
  const double t = mul(m, kd);
  const double margin = mul(fabs(a), 0x1.0p-50);
  if (!(fabs(a) >= 0x1.0p-900)) return m > dvd(a, kd);  // margin would underflow
  if (t > add(a, margin)) return true;
  if (t < sub(a, margin)) return false;
  return m > dvd(a, kd);
}

// Exact emulation of the reference's sequential cumulative sum (prox.cpp:44-51) over the
// sorted candidates c[0..L) (descending, >= 0), fused with its break test.  While the
// running sum S stays inside one binade [2^e, 2^(e+1)), every fl(S + m) is S plus m rounded
// to the fixed grid u = 2^(e-52) (round-to-nearest), so the prefix sums of an epoch are one
// exact integer prefix scan of grid counts.  The first position whose sum leaves the binade,
// or whose rounding is a tie (decided by the parity of S), is done as one IEEE addition and
// starts the next epoch.  The short epochs at the top are done by a sequential prologue;
// later epochs scan windows whose size follows the (doubling) epoch lengths.
// Returns the first failing index ff (L if none) and S_{ff-1} (the sum whose candidate is
// theta).  All threads of the block call it and receive the same result.
struct ScanShared {
  long long wsum[L1G_PREFIX_PT / 32];
  long long ev[L1G_PREFIX_PT / 32][2];
  double sv[L1G_PREFIX_PT];
  double pro[2];
  long long pro_i;
};

constexpr int PREFIX_PROLOGUE = 64;

__device__ long long prefix_break(const double* c, long long L, double rho, ScanShared& ss,
                                  double* s_before) {
  constexpr int NT = L1G_PREFIX_PT;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr long long TWO53 = 1LL << 53;
  // ---- sequential prologue (thread 0): S_0 = fl(0 + c_0) = c_0, then IEEE additions
  if (tid == 0) {
    const long long lim = L < PREFIX_PROLOGUE ? L : PREFIX_PROLOGUE;
    double S = 0.0, prev = 0.0;
    long long i = 0, ff = -1;
    for (; i < lim; ++i) {
      prev = S;
      S = add(S, c[i]);
      if (!passes(c[i], S, rho, i + 1)) {
        ff = i;
        break;
      }
    }
    ss.pro_i = ff >= 0 ? -(ff + 1) : lim;  // <0: failure at -(pro_i)-1
    ss.pro[0] = ff >= 0 ? prev : S;
  }
  __syncthreads();
  const long long pi = ss.pro_i;
  double S_prev = ss.pro[0];
  __syncthreads();
  if (pi < 0) {
    *s_before = S_prev;
    return -pi - 1;
  }
  long long i0 = pi;
  long long window = NT;
  while (i0 < L) {
    if (!(S_prev >= 0x1.0p-960)) {  // (sub)tiny running sum: plain scalar step, uniform
      const double S = add(S_prev, c[i0]);
      if (!passes(c[i0], S, rho, i0 + 1)) {
        *s_before = S_prev;
        return i0;
      }
      S_prev = S;
      ++i0;
      continue;
    }
    const long long n = (L - i0) < window ? (L - i0) : window;
    const long long E = (n + NT - 1) / NT;
    const long long wend = i0 + n;
    const long long p0 = i0 + (long long)tid * E;
    const long long p1 = p0 + E < wend ? p0 + E : wend;
    const long long ebits = (__double_as_longlong(S_prev) >> 52) & 0x7ff;
    const double u = __longlong_as_double((ebits - 52) << 52);           // 2^(e-52)
    const double inv_u = __longlong_as_double((2098 - ebits) << 52);    // 2^(52-e)
    const double hu = 0.5 * u;
    const long long base_q = (long long)(S_prev * inv_u);               // exact, < 2^53
    // pass 1: grid counts of my positions
    long long tot = 0;
    for (long long i = p0; i < p1; ++i) {
      const double m = c[i];
      const double qd = floor(m * inv_u);
      tot += (long long)qd + (sub(m, qd * u) > hu ? 1 : 0);
    }
    long long inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) ss.wsum[warp] = inc;
    __syncthreads();
    long long off = inc - tot, btot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const long long x = ss.wsum[w];
      off += w < warp ? x : 0;
      btot += x;
    }
    // pass 2: exact sums and tests up to my first event (failure or binade exit / tie)
    long long P = off, my_ff = LLONG_MAX, my_fb = LLONG_MAX;
    for (long long i = p0; i < p1; ++i) {
      const double m = c[i];
      const double qd = floor(m * inv_u);
      const double r = sub(m, qd * u);
      const long long q = (long long)qd + (r > hu ? 1 : 0);
      if (r == hu || base_q + P + q >= TWO53) {
        my_fb = i;
        ss.sv[tid] = i == i0 ? S_prev : (double)(base_q + P) * u;  // S_{i-1}
        break;
      }
      P += q;
      if (!passes(m, (double)(base_q + P) * u, rho, i + 1)) {
        my_ff = i;
        ss.sv[tid] = i == i0 ? S_prev : (double)(base_q + P - q) * u;  // S_{i-1}
        break;
      }
    }
    long long a0 = my_ff, a1 = my_fb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 = min(a0, __shfl_xor_sync(0xffffffffu, a0, o));
      a1 = min(a1, __shfl_xor_sync(0xffffffffu, a1, o));
    }
    if (lane == 0) {
      ss.ev[warp][0] = a0;
      ss.ev[warp][1] = a1;
    }
    __syncthreads();
    long long FF = LLONG_MAX, FB = LLONG_MAX;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      FF = min(FF, ss.ev[w][0]);
      FB = min(FB, ss.ev[w][1]);
    }
    if (FF < FB) {  // a failure inside the exact range
      *s_before = ss.sv[(FF - i0) / E];
      __syncthreads();
      return FF;
    }
    if (FB == LLONG_MAX) {  // the whole window is exact and passes: same epoch continues
      S_prev = (double)(base_q + btot) * u;
      i0 = wend;
      window *= 2;
      __syncthreads();
      continue;
    }
    // one IEEE addition at the first binade exit / tie, evaluated by every thread alike
    const double Sm1 = ss.sv[(FB - i0) / E];
    __syncthreads();
    const double S = add(Sm1, c[FB]);
    if (!passes(c[FB], S, rho, FB + 1)) {
      *s_before = Sm1;
      return FB;
    }
    // the next epoch is about as long as the whole prefix so far: size the window for it
    const long long len = FB + 1;
    window = ((len + NT - 1) / NT) * NT;
    S_prev = S;
    i0 = FB + 1;
  }
  *s_before = S_prev;
  return L;
}

}  // namespace l1g
