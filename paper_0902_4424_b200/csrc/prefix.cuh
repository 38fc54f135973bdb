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

#ifdef L1G_PREFIX_STAMPS  // sub-epoch clock stamps (tools/bench_prefix.cu)
#define L1G_PSTAMP(k) \
  if (threadIdx.x == 0 && ntr > 0 && ntr <= 64) L1G_PREFIX_STAMPS[(ntr - 1) * 8 + (k)] = clock64();
#define L1G_HSTAMP(k) \
  if (threadIdx.x == 0) L1G_PREFIX_STAMPS[64 * 8 + (k)] = clock64();
#else
#define L1G_PSTAMP(k)
#define L1G_HSTAMP(k)
#endif

#ifndef L1G_PREFIX_HEAD
#define L1G_PREFIX_HEAD 256
#endif
constexpr int PREFIX_HEAD = L1G_PREFIX_HEAD;
constexpr int PREFIX_MAXW = 32;  // warps per block

// A run of positions as a function of the parity of the running grid count N it starts
// from: a rounding tie (m an odd multiple of half a grid step) rounds N + q + 1/2 to the
// even neighbour, so it adds q or q + 1 depending on N's parity and always leaves N even;
// other positions add their fixed q.  d0 / p0: increment and final parity from an even
// start; from an odd start the increment is d0 + dl (dl in {-1, 0, 1}) and the final parity
// p1.  Composition is associative, so ties ride along the prefix scan.
struct ParSeg {
  long long d0;
  int dl, p0, p1;
};
__device__ __forceinline__ ParSeg seg_id() { return ParSeg{0, 0, 0, 1}; }
__device__ __forceinline__ ParSeg seg_then(const ParSeg& A, const ParSeg& B) {
  ParSeg C;
  const int b0 = A.p0 ? B.dl : 0, b1 = A.p1 ? B.dl : 0;
  C.d0 = A.d0 + B.d0 + b0;
  C.dl = A.dl + b1 - b0;
  C.p0 = A.p0 ? B.p1 : B.p0;
  C.p1 = A.p1 ? B.p1 : B.p0;
  return C;
}
// one position: grid count q, tie or not
__device__ __forceinline__ ParSeg seg_elem(long long q, bool tie) {
  const int odd = (int)(q & 1);
  if (!tie) return ParSeg{q, 0, odd, odd ^ 1};
  return ParSeg{q + odd, odd ? -1 : 1, 0, 0};
}
// the running count after the segment, from the concrete count N
__device__ __forceinline__ long long seg_apply(const ParSeg& s, long long N) {
  return N + s.d0 + ((N & 1) ? s.dl : 0);
}
__device__ __forceinline__ int seg_pack(const ParSeg& v) {
  return (v.dl + 1) | (v.p0 << 2) | (v.p1 << 3);
}
__device__ __forceinline__ ParSeg seg_unpack(long long d0, int pk) {
  return ParSeg{d0, (pk & 3) - 1, (pk >> 2) & 1, (pk >> 3) & 1};
}
__device__ __forceinline__ ParSeg seg_shfl_up(const ParSeg& v, int o) {
  return seg_unpack(__shfl_up_sync(0xffffffffu, v.d0, o),
                    __shfl_up_sync(0xffffffffu, seg_pack(v), o));
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

struct ScanShared {
  alignas(16) double head[PREFIX_HEAD];
  long long wd0[2][PREFIX_MAXW];  // warp segments (double-buffered by epoch parity)
  int wpk[2][PREFIX_MAXW];
  int epos[2][PREFIX_MAXW];       // per warp: first event (position, kind, count before)
  int ekind[2][PREFIX_MAXW];
  long long en[2][PREFIX_MAXW];
  long long fq[2][PREFIX_MAXW];   // fast path: warp sums of grid counts, any tie in the warp
  int ftie[2][PREFIX_MAXW];
  int hbad[PREFIX_MAXW];
  int epochs;  // telemetry: windows scanned by the last call
};

// The reference's sequential cumulative sum over head[0..H) in place (head is PREFIX_HEAD
// long, zero past H): one thread, vector loads one batch ahead, each sum in its own register.
__device__ __forceinline__ void head_sums(double* head, int H) {
  double2* hp = reinterpret_cast<double2*>(head);
  double run = 0.0;
  double2 v[4], w[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) v[u] = hp[u];
  for (int i0 = 0; i0 < H; i0 += 8) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      w[u] = i0 + 8 < PREFIX_HEAD ? hp[(i0 + 8) / 2 + u] : make_double2(0.0, 0.0);
    double hs[8];
    hs[0] = add(run, v[0].x);
    hs[1] = add(hs[0], v[0].y);
#pragma unroll
    for (int u = 1; u < 4; ++u) {
      hs[2 * u] = add(hs[2 * u - 1], v[u].x);
      hs[2 * u + 1] = add(hs[2 * u], v[u].y);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) hp[i0 / 2 + u] = make_double2(hs[2 * u], hs[2 * u + 1]);
    run = hs[7];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = w[u];
  }
}

// Exact emulation of the reference's sequential cumulative sum (prox.cpp:44-51) over the
// sorted candidates c[0..L) (descending, >= 0), fused with its break test.  While the
// running sum S stays inside one binade [2^e, 2^(e+1)), every fl(S + m) is S plus m rounded
// to the fixed grid u = 2^(e-52) (round-to-nearest), so the prefix sums of an epoch are one
// exact integer prefix scan of grid counts (computed from the mantissa bits; rounding ties,
// decided by the parity of the running count, ride along the scan as parity-dependent
// segments).  The first position whose sum leaves the binade is done as one IEEE addition
// and starts the next epoch.  The short epochs at the top are cheaper as the reference's
// own sequential sum (one dependent add per position); after PREFIX_HEAD positions the
// block scans windows sized to the (doubling) epochs.  Returns the first failing index ff
// (L if none) and S_{ff-1} (the sum whose candidate is theta).  All NT threads of the block
// call it and receive the same result.
template <int NT = 512>
__device__ long long prefix_break(const double* c, long long Ll, double rho, ScanShared& ss,
                                  double* s_before) {
  static_assert(NT % 32 == 0 && NT <= 32 * PREFIX_MAXW &&
                    (PREFIX_HEAD % NT == 0 || NT % PREFIX_HEAD == 0),
                "prefix_break block shape");
  // the first NT threads of the block run it: a block barrier, or a named one for fewer
  auto bsync = [] {
    if constexpr (NT == 512) __syncthreads();
    else named_bar_sync(3, NT);
  };
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr long long TWO53 = 1LL << 53;
  constexpr unsigned FULL = 0xffffffffu;
  const int L = (int)Ll;
  if (L <= 0) {
    *s_before = 0.0;
    return 0;
  }
  // ---- head: warp 0 stages c[0..H) in shared memory, one thread adds sequentially (vector
  //      loads one batch ahead, each sum in its own register), then every thread tests one
  //      position
  const int H = L < PREFIX_HEAD ? L : PREFIX_HEAD;
  L1G_HSTAMP(0)
  if (warp == 0) {
    for (int i = lane; i < PREFIX_HEAD; i += 32) ss.head[i] = i < H ? c[i] : 0.0;
    __syncwarp();
    if (lane == 0) head_sums(ss.head, H);
  }
  L1G_HSTAMP(1)
  bsync();
  {
    int first = INT_MAX;
#pragma unroll
    for (int i0 = 0; i0 < PREFIX_HEAD; i0 += NT) {  // every thread tests positions tid, tid + NT, ..
      const int i = i0 + tid;
      const bool bad = i < H && !passes(c[i], ss.head[i], rho, i + 1);
      const unsigned bb = __ballot_sync(FULL, bad);
      if (first == INT_MAX && bb) first = i0 + warp * 32 + __ffs(bb) - 1;
    }
    if (lane == 0) ss.hbad[warp] = first;
  }
  L1G_HSTAMP(2)
  bsync();
  L1G_HSTAMP(3)
  {
    int ff = INT_MAX;
#pragma unroll
    for (int w = 0; w < NW; ++w) ff = min(ff, ss.hbad[w]);
    if (ff != INT_MAX || H == L) {
      if (tid == 0) ss.epochs = 0;
      *s_before = ff == INT_MAX ? ss.head[H - 1] : (ff > 0 ? ss.head[ff - 1] : 0.0);
      return ff == INT_MAX ? L : ff;
    }
  }
  double S_prev = ss.head[H - 1];
  int i0 = H, window = 2 * H, par = 0;
#ifdef L1G_PREFIX_TRACE
  int ntr = 0;
#endif
  int nep = 0;
  while (i0 < L) {
    ++nep;
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
        if (tid == 0) ss.epochs = nep;
        return i0;
      }
      S_prev = S;
      ++i0;
      continue;
    }
    const int n = (L - i0) < window ? (L - i0) : window;
    const int E = (n + NT - 1) / NT;
    const int wend = i0 + n;
    const int p0 = min(i0 + tid * E, wend);
    const int p1 = min(p0 + E, wend);
    const long long sbits = __double_as_longlong(S_prev);
    const int be = (int)(sbits >> 52);
    const long long base_q = (sbits & ((1LL << 52) - 1)) | (1LL << 52);  // S_prev / u
    // pass 1: grid counts of this thread's run.  Rounding ties are rare; without any in the
    // window the running counts are a plain integer prefix sum (one int64 warp scan and the
    // 16 warp totals), with one the parity segments below decide them
    long long qs = 0;
    bool anytie = false;
#pragma unroll 4
    for (int i = p0; i < p1; ++i) {
      bool t;
      qs += grid_count(c[i], be, &t);
      anytie |= t;
    }
    const unsigned tball = __ballot_sync(FULL, anytie);
    long long qinc = qs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, qinc, o);
      if (lane >= o) qinc += y;
    }
    if (lane == 31) {
      ss.fq[par][warp] = qinc;
      ss.ftie[par][warp] = tball != 0;
    }
    L1G_PSTAMP(0)
    bsync();
    L1G_PSTAMP(1)
    long long N, Nend;
    {
      long long wex = 0, tot = 0;
      int ties = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const long long d = ss.fq[par][w];
        wex += w < warp ? d : 0;
        tot += d;
        ties |= ss.ftie[par][w];
      }
      N = base_q + wex + (qinc - qs);
      Nend = base_q + tot;
      if (ties) {  // uniform over the block: the parity-segment scan
        ParSeg me = seg_id();
#pragma unroll 4
        for (int i = p0; i < p1; ++i) {
          bool t;
          const long long q = grid_count(c[i], be, &t);
          me = seg_then(me, seg_elem(q, t));
        }
        const ParSeg incl = seg_warp_scan(me, lane);
        if (lane == 31) {
          ss.wd0[par][warp] = incl.d0;
          ss.wpk[par][warp] = seg_pack(incl);
        }
        bsync();
        // concrete counts: the warps' starts by applying the warp segments in order (the
        // parity chain is a 1-bit select per warp; increments add up independently)
        long long Nw = base_q, accd = base_q;
        int accl = 0, pb = (int)(base_q & 1);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const long long d0 = ss.wd0[par][w];
          const int pk = ss.wpk[par][w];
          Nw = w == warp ? accd + accl : Nw;
          accl += pb ? (pk & 3) - 1 : 0;
          accd += d0;
          pb = pb ? (pk >> 3) & 1 : (pk >> 2) & 1;
        }
        Nend = accd + accl;
        ParSeg ex = seg_shfl_up(incl, 1);
        if (lane == 0) ex = seg_id();
        N = seg_apply(ex, Nw);
      }
    }
    L1G_PSTAMP(2)
    // pass 2: exact sums and tests; my first event (1 failure, 2 binade exit,
    // 3 test too close to call), branch-free so positions overlap
    int my_ev = INT_MAX, kind = 0;
    long long my_n = 0;
    double kd = (double)(p0 + 1);
#pragma unroll 4
    for (int i = p0; i < p1; ++i) {
      const double m = c[i];
      bool tie;
      const long long q = grid_count(m, be, &tie);
      const long long Nn = N + q + (tie ? ((N + q) & 1) : 0);
      const int stt = Nn >= TWO53 ? 2 : quick_test(m, from_grid(Nn, be), rho, kd);
      const bool take = stt != 0 && my_ev == INT_MAX;
      my_ev = take ? i : my_ev;
      kind = take ? stt : kind;
      my_n = take ? N : my_n;
      N = Nn;
      kd = add(kd, 1.0);
    }
    L1G_PSTAMP(3)
    // first event of the window: per warp (positions increase with the lane), then over
    // the warps in order
    const unsigned have = __ballot_sync(FULL, my_ev != INT_MAX);
    if (have) {
      if (lane == __ffs(have) - 1) {
        ss.epos[par][warp] = my_ev;
        ss.ekind[par][warp] = kind;
        ss.en[par][warp] = my_n;
      }
    } else if (lane == 0) {
      ss.epos[par][warp] = INT_MAX;
    }
    bsync();
    int ew = -1;
#pragma unroll
    for (int w = NW - 1; w >= 0; --w) ew = ss.epos[par][w] != INT_MAX ? w : ew;
    L1G_PSTAMP(4)
    if (ew < 0) {  // the whole window is exact and passes: the epoch continues
      S_prev = from_grid(Nend, be);
      i0 = wend;
      window *= 2;
      par ^= 1;
      continue;
    }
    const int ev = ss.epos[par][ew], evk = ss.ekind[par][ew];
    const long long nb = ss.en[par][ew];
    par ^= 1;
#ifdef L1G_PREFIX_TRACE
    if (threadIdx.x == 0 && ntr > 0 && ntr <= 64) L1G_PREFIX_TRACE[3 * (ntr - 1) + 2] += 1000000LL * evk;
#endif
    const double sb = from_grid(nb, be);  // S_{ev-1}
    if (evk == 1) {
      *s_before = sb;
      if (tid == 0) ss.epochs = nep;
      return ev;
    }
    if (evk == 3) {  // exact test with the division; on success the epoch goes on
      bool t;
      const long long qe = grid_count(c[ev], be, &t);
      const double Se = from_grid(nb + qe + (t ? ((nb + qe) & 1) : 0), be);
      if (!passes(c[ev], Se, rho, ev + 1)) {
        *s_before = sb;
        if (tid == 0) ss.epochs = nep;
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
      if (tid == 0) ss.epochs = nep;
      return ev;
    }
    L1G_PSTAMP(5)
    // the running sum doubles again after a bit more than the prefix so far (candidates
    // decrease): size the window to twice the prefix, overshooting rather than re-scanning
    window = ((2 * (ev + 1) + 31) >> 5) << 5;
    S_prev = S;
    i0 = ev + 1;
  }
  *s_before = S_prev;
  if (tid == 0) ss.epochs = nep;
  return L;
}

}  // namespace l1g
