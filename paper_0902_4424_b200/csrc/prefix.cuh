// prefix.cuh -- exact parallel emulation of a sequential floating-point cumulative sum
// (the sort-and-scan threshold of prox.cpp:43-52), used by project.cu.
#pragma once
#include "common.cuh"

namespace l1g {


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


// Grid count of m >= 0 on the grid of a running sum with biased exponent be (m <= sum):
// q = round(m / u), u = 2^(be - 1075), by integer shifts of the mantissa; tie = exact half.
__device__ __forceinline__ long long grid_count(double m, int be, bool* tie) {
  const long long bits = __double_as_longlong(m);
  const int bm = (int)(bits >> 52);
  const long long M = (bits & ((1LL << 52) - 1)) | (1LL << 52);
  const int sh = be - bm;
  const int s1 = sh < 1 ? 1 : (sh > 62 ? 62 : sh);
  const long long rem = M & ((1LL << s1) - 1), half = 1LL << (s1 - 1);
  const long long q = (M >> s1) + (rem > half ? 1 : 0);
  // bm == 0: zero or subnormal, far below half a grid step; sh > 53: below half a step
  const bool zero = bm == 0 || sh > 53;
  *tie = !zero && sh > 0 && rem == half;
  return zero ? 0 : (sh == 0 ? M : q);
}
// The break test without the division, for a scan: 0 pass, 1 fail, 3 too close to call
// (resolved afterwards by passes()).
__device__ __forceinline__ int quick_test(double m, double S, double rho, double kd) {
  const double a = sub(S, rho);
  const double t = mul(m, kd);
  const double margin = mul(fabs(a), 0x1.0p-50);
  const bool tiny = !(fabs(a) >= 0x1.0p-900);
  const bool ps = t > add(a, margin), fl = t < sub(a, margin);
  return tiny ? 3 : (ps ? 0 : (fl ? 1 : 3));
}
// the double N * 2^(be - 1075) for N in [2^52, 2^53)
__device__ __forceinline__ double from_grid(long long N, int be) {
  return __longlong_as_double(((long long)(be - 1) << 52) + N);
}

constexpr int PREFIX_HEAD = 256;
constexpr int PREFIX_MAXW = 32;  // warps per block

struct ScanShared {
  double head[PREFIX_HEAD];
  long long wsum[PREFIX_MAXW];
  long long wd0[PREFIX_MAXW], wd1[PREFIX_MAXW];
  int wp[PREFIX_MAXW];
  long long wev[PREFIX_MAXW];
  long long ev, nb;
  int kind;
  double sb;
  int epochs;  // telemetry: windows scanned by the last call
};

// A run of positions as a function of the parity of the running grid count N it starts
// from: a rounding tie (m an odd multiple of half a grid step) rounds N + q + 1/2 to the
// even neighbour, so it adds q or q + 1 depending on N's parity and always leaves N even;
// other positions add their fixed q.  (d0, p0) / (d1, p1): increment and final parity for
// an even / odd start.  Composition is associative, so ties ride along the prefix scan.
struct ParSeg {
  long long d0, d1;
  int p0, p1;
};
__device__ __forceinline__ ParSeg seg_then(const ParSeg& A, const ParSeg& B) {
  ParSeg C;
  C.d0 = A.d0 + (A.p0 ? B.d1 : B.d0);
  C.p0 = A.p0 ? B.p1 : B.p0;
  C.d1 = A.d1 + (A.p1 ? B.d1 : B.d0);
  C.p1 = A.p1 ? B.p1 : B.p0;
  return C;
}
__device__ __forceinline__ ParSeg seg_shfl_up(const ParSeg& v, int o) {
  ParSeg r;
  r.d0 = __shfl_up_sync(0xffffffffu, v.d0, o);
  r.d1 = __shfl_up_sync(0xffffffffu, v.d1, o);
  const int pk = __shfl_up_sync(0xffffffffu, v.p0 | (v.p1 << 1), o);
  r.p0 = pk & 1;
  r.p1 = pk >> 1;
  return r;
}
__device__ __forceinline__ ParSeg seg_shfl(const ParSeg& v, int src) {
  ParSeg r;
  r.d0 = __shfl_sync(0xffffffffu, v.d0, src);
  r.d1 = __shfl_sync(0xffffffffu, v.d1, src);
  const int pk = __shfl_sync(0xffffffffu, v.p0 | (v.p1 << 1), src);
  r.p0 = pk & 1;
  r.p1 = pk >> 1;
  return r;
}
// inclusive scan of per-lane segments over the warp (earlier lanes first)
__device__ __forceinline__ ParSeg seg_warp_scan(ParSeg v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const ParSeg y = seg_shfl_up(v, o);
    if (lane >= o) v = seg_then(y, v);
  }
  return v;
}

// Exact emulation of the reference's sequential cumulative sum (prox.cpp:44-51) over the
// sorted candidates c[0..L) (descending, >= 0), fused with its break test.  While the
// running sum S stays inside one binade [2^e, 2^(e+1)), every fl(S + m) is S plus m rounded
// to the fixed grid u = 2^(e-52) (round-to-nearest), so the prefix sums of an epoch are one
// exact integer prefix scan of grid counts (computed from the mantissa bits; rounding ties,
// decided by the parity of the running count, ride along the scan as parity-dependent
// segments).  The first position whose sum leaves the binade is done as one IEEE addition
// and starts the next epoch.  The short epochs at the
// top are cheaper as the reference's own sequential sum (one dependent add per position);
// after PREFIX_HEAD positions the block scans windows sized to the (doubling) epochs.
// Returns the first failing index ff (L if none) and S_{ff-1} (the sum whose candidate is
// theta).  All threads of the block call it (blockDim a multiple of 32, <= 1024) and
// receive the same result.
__device__ long long prefix_break(const double* c, long long L, double rho, ScanShared& ss,
                                  double* s_before) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  constexpr long long TWO53 = 1LL << 53;
  constexpr unsigned FULL = 0xffffffffu;
  if (L <= 0) {
    *s_before = 0.0;
    return 0;
  }
  // ---- head: lane 0 of warp 0 adds sequentially, warp 0 tests in parallel
  const long long H = L < PREFIX_HEAD ? L : PREFIX_HEAD;
  if (warp == 0) {
    if (lane == 0) {
      double run = 0.0, v[8], w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = u < H ? c[u] : 0.0;
      for (long long i0 = 0; i0 < H; i0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = i0 + 8 + u < H ? c[i0 + 8 + u] : 0.0;  // next batch
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0 + u < H) {
            run = add(run, v[u]);
            ss.head[i0 + u] = run;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = w[u];
      }
    }
    __syncwarp();
    long long ff = LLONG_MAX;
    for (long long i = lane; i - lane < H; i += 32) {
      const bool ok = i < H ? passes(c[i], ss.head[i], rho, i + 1) : true;
      const unsigned bad = __ballot_sync(FULL, !ok);
      if (bad) {
        ff = i - lane + (__ffs(bad) - 1);
        break;
      }
    }
    if (lane == 0) {
      ss.ev = ff;
      ss.sb = ff == LLONG_MAX ? ss.head[H - 1] : (ff > 0 ? ss.head[ff - 1] : 0.0);
    }
  }
  __syncthreads();
  {
    const long long ff = ss.ev;
    const double sb = ss.sb;
    __syncthreads();
    if (ff != LLONG_MAX) {
      *s_before = sb;
      return ff;
    }
    if (H == L) {
      *s_before = sb;
      return L;
    }
  }
  double S_prev = ss.head[H - 1];
  long long i0 = H, window = 2 * H;
#ifdef L1G_PREFIX_TRACE
  int ntr = 0;
#endif
  if (threadIdx.x == 0) ss.epochs = 0;
  while (i0 < L) {
    if (threadIdx.x == 0) ++ss.epochs;
#ifdef L1G_PREFIX_TRACE
    if (threadIdx.x == 0 && ntr < 64) {
      L1G_PREFIX_TRACE[3 * ntr] = clock64();
      L1G_PREFIX_TRACE[3 * ntr + 1] = i0;
      L1G_PREFIX_TRACE[3 * ntr + 2] = window;
      ++ntr;
    }
#endif
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
    const long long sbits = __double_as_longlong(S_prev);
    const int be = (int)(sbits >> 52);
    const long long base_q = (sbits & ((1LL << 52) - 1)) | (1LL << 52);  // S_prev / u
    // pass 1: grid counts of my positions (a tie counted at its floor)
    long long tot = 0;
    int tie_here = 0;
#pragma unroll 4
    for (long long i = p0; i < p1; ++i) {
      bool t;
      tot += grid_count(c[i], be, &t);
      tie_here |= t;
    }
    long long inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) ss.wsum[warp] = inc;
    const int any_tie = __syncthreads_or(tie_here);
    const int par0 = (int)(base_q & 1);
    long long start, btot;
    if (!any_tie) {  // warp totals: inclusive scan over the warps by shuffles
      const long long x = lane < NW ? ss.wsum[lane] : 0;
      long long sc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(FULL, sc, o);
        if (lane >= o) sc += y;
      }
      btot = __shfl_sync(FULL, sc, 31);
      start = inc - tot + (warp > 0 ? __shfl_sync(FULL, sc, warp - 1) : 0);
    } else {  // rounding ties in the window: scan parity-dependent segments instead
      ParSeg me = {0, 0, 0, 1};
      for (long long i = p0; i < p1; ++i) {
        bool tie;
        const long long q = grid_count(c[i], be, &tie);
        if (!tie) {
          me.d0 += q;
          me.d1 += q;
          me.p0 ^= (int)(q & 1);
          me.p1 ^= (int)(q & 1);
        } else {
          me.d0 += q + ((me.p0 + q) & 1);
          me.d1 += q + ((me.p1 + q) & 1);
          me.p0 = 0;
          me.p1 = 0;
        }
      }
      const ParSeg incl = seg_warp_scan(me, lane);
      if (lane == 31) {
        ss.wd0[warp] = incl.d0;
        ss.wd1[warp] = incl.d1;
        ss.wp[warp] = incl.p0 | (incl.p1 << 1);
      }
      __syncthreads();
      ParSeg t = {0, 0, 0, 1};
      if (lane < NW) {
        t.d0 = ss.wd0[lane];
        t.d1 = ss.wd1[lane];
        t.p0 = ss.wp[lane] & 1;
        t.p1 = ss.wp[lane] >> 1;
      }
      const ParSeg ti = seg_warp_scan(t, lane);
      const ParSeg total = seg_shfl(ti, 31);
      const ParSeg wx = seg_shfl(ti, warp > 0 ? warp - 1 : 0);
      const ParSeg wpre = warp > 0 ? wx : ParSeg{0, 0, 0, 1};
      ParSeg lx = seg_shfl_up(incl, 1);
      if (lane == 0) lx = ParSeg{0, 0, 0, 1};
      const ParSeg before = seg_then(wpre, lx);
      btot = par0 ? total.d1 : total.d0;
      start = par0 ? before.d1 : before.d0;
    }
    // pass 2: exact sums and tests; my first event (1 failure, 2 binade exit,
    // 3 test too close to call), branch-free so positions overlap
    long long N = base_q + start, my_ev = LLONG_MAX, my_n = 0;
    int kind = 0;
    double kd = (double)(p0 + 1);
#pragma unroll 4
    for (long long i = p0; i < p1; ++i) {
      const double m = c[i];
      bool tie;
      const long long q = grid_count(m, be, &tie);
      const long long Nn = N + q + (tie ? ((N + q) & 1) : 0);
      const int stt = Nn >= TWO53 ? 2 : quick_test(m, from_grid(Nn, be), rho, kd);
      const bool take = stt != 0 && my_ev == LLONG_MAX;
      my_ev = take ? i : my_ev;
      kind = take ? stt : kind;
      my_n = take ? N : my_n;
      N = Nn;
      kd = add(kd, 1.0);
    }
    // first event of the window (positions increase with the thread index)
    const unsigned have = __ballot_sync(FULL, my_ev != LLONG_MAX);
    if (lane == 0) ss.wev[warp] = have ? (long long)warp * 32 + (__ffs(have) - 1) : LLONG_MAX;
    __syncthreads();
    long long owner = lane < NW ? ss.wev[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) owner = min(owner, __shfl_xor_sync(FULL, owner, o));
    if (owner == LLONG_MAX) {  // the whole window is exact and passes: the epoch continues
      S_prev = from_grid(base_q + btot, be);
      i0 = wend;
      window *= 2;
      __syncthreads();
      continue;
    }
    if (tid == owner) {
      ss.ev = my_ev;
      ss.kind = kind;
      ss.nb = my_n;
    }
    __syncthreads();
    const long long ev = ss.ev, nb = ss.nb;
    const int evk = ss.kind;
    __syncthreads();
#ifdef L1G_PREFIX_TRACE
    if (threadIdx.x == 0 && ntr > 0 && ntr <= 64) L1G_PREFIX_TRACE[3 * (ntr - 1) + 2] += 1000000LL * evk;
#endif
    const double sb = from_grid(nb, be);  // S_{ev-1}
    if (evk == 1) {
      *s_before = sb;
      return ev;
    }
    if (evk == 3) {  // exact test with the division; on success the epoch goes on
      bool t;
      const long long qe = grid_count(c[ev], be, &t);
      const double Se = from_grid(nb + qe + (t ? ((nb + qe) & 1) : 0), be);
      if (!passes(c[ev], Se, rho, ev + 1)) {
        *s_before = sb;
        return ev;
      }
      S_prev = Se;
      i0 = ev + 1;
      continue;
    }
    // one IEEE addition at the binade exit, evaluated by every thread alike
    const double S = add(sb, c[ev]);
    if (!passes(c[ev], S, rho, ev + 1)) {
      *s_before = sb;
      return ev;
    }
    // the running sum doubles again after a bit more than the prefix so far (candidates
    // decrease): size the window to twice the prefix, overshooting rather than re-scanning
    window = ((2 * (ev + 1) + 31) >> 5) << 5;
    S_prev = S;
    i0 = ev + 1;
  }
  *s_before = S_prev;
  return L;
}

}  // namespace l1g
