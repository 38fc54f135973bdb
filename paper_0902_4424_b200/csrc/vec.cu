// vec.cu -- operator construction (tiling, on-device generators), canonical vector
// reductions and small element-wise / scalar kernels used outside the hot loop.
#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"
#include "vec.h"

namespace l1g {

// ---------------------------------------------------------------- deterministic normals
// Philox4x32-10 + Box-Muller from IEEE basic operations only; bit-identical to
// oracle/l1oracle.c (orc_philox4x32, orc_det_log, orc_det_sincos2pi, normal_pair).
__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
  const uint64_t v = ((uint64_t)hi << 32) | lo;
  return mul((double)(v >> 11), 0x1.0p-53);
}

__device__ double det_log(double u) {
  uint64_t bits = (uint64_t)__double_as_longlong(u);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  bits = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m = __longlong_as_double((long long)bits);
  if (m > 1.4142135623730951) {
    m = mul(m, 0.5);
    e += 1;
  }
  const double s = dvd(sub(m, 1.0), add(m, 1.0));
  const double s2 = mul(s, s);
  double q = 1.0 / 25.0;
  q = add(mul(q, s2), 1.0 / 23.0);
  q = add(mul(q, s2), 1.0 / 21.0);
  q = add(mul(q, s2), 1.0 / 19.0);
  q = add(mul(q, s2), 1.0 / 17.0);
  q = add(mul(q, s2), 1.0 / 15.0);
  q = add(mul(q, s2), 1.0 / 13.0);
  q = add(mul(q, s2), 1.0 / 11.0);
  q = add(mul(q, s2), 1.0 / 9.0);
  q = add(mul(q, s2), 1.0 / 7.0);
  q = add(mul(q, s2), 1.0 / 5.0);
  q = add(mul(q, s2), 1.0 / 3.0);
  const double logm = add(mul(2.0, s), mul(mul(2.0, s), mul(s2, q)));
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  return add(mul((double)e, ln2_hi), add(mul((double)e, ln2_lo), logm));
}

__device__ void det_sincos2pi(double u, double* so, double* co) {
  const double fq = floor(add(mul(4.0, u), 0.5));
  const int q = (int)fq;
  const double r = sub(u, mul(fq, 0.25));
  const double t = mul(r, 6.283185307179586);
  const double t2 = mul(t, t);
  double ps = -1.0 / 121645100408832000.0;
  ps = add(mul(ps, t2), 1.0 / 355687428096000.0);
  ps = sub(mul(ps, t2), 1.0 / 1307674368000.0);
  ps = add(mul(ps, t2), 1.0 / 6227020800.0);
  ps = sub(mul(ps, t2), 1.0 / 39916800.0);
  ps = add(mul(ps, t2), 1.0 / 362880.0);
  ps = sub(mul(ps, t2), 1.0 / 5040.0);
  ps = add(mul(ps, t2), 1.0 / 120.0);
  ps = sub(mul(ps, t2), 1.0 / 6.0);
  const double sn = add(t, mul(t, mul(t2, ps)));
  double pc = 1.0 / 6402373705728000.0;
  pc = sub(mul(pc, t2), 1.0 / 20922789888000.0);
  pc = add(mul(pc, t2), 1.0 / 87178291200.0);
  pc = sub(mul(pc, t2), 1.0 / 479001600.0);
  pc = add(mul(pc, t2), 1.0 / 3628800.0);
  pc = sub(mul(pc, t2), 1.0 / 40320.0);
  pc = add(mul(pc, t2), 1.0 / 720.0);
  pc = sub(mul(pc, t2), 1.0 / 24.0);
  pc = add(mul(pc, t2), 0.5);
  const double cs = sub(1.0, mul(t2, pc));
  switch (q & 3) {
    case 0: *so = sn; *co = cs; break;
    case 1: *so = cs; *co = -sn; break;
    case 2: *so = -sn; *co = -cs; break;
    default: *so = -cs; *co = sn; break;
  }
}

__device__ double det_normal(uint64_t seed, uint32_t stream, uint64_t index) {
  const uint64_t pair = index >> 1;
  uint32_t c[4] = {(uint32_t)pair, (uint32_t)(pair >> 32), stream, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u1 = sub(1.0, u53(c[0], c[1]));
  const double u2 = u53(c[2], c[3]);
  const double radius = __dsqrt_rn(mul(-2.0, det_log(u1)));
  double sn, cs;
  det_sincos2pi(u2, &sn, &cs);
  return (index & 1u) ? mul(radius, sn) : mul(radius, cs);
}

// ---------------------------------------------------------------- operator construction
// One CTA per tile (grid-stride): the source is read in its natural order (row-major tile
// rows, or column-major runs when COLREAD), staged in shared memory, and the tile is written
// out as one contiguous coalesced 16 KB run in the tiled layout (common.cuh).
template <bool COLREAD, class F>
__global__ void __launch_bounds__(256) fill_tiled_kernel(double* K, int64_t ntiles, int64_t ncb,
                                                         int64_t n, int64_t p, int64_t row0, F val) {
  __shared__ double t[TR * (TC + 1)];  // row-major staging, padded: conflict-free both ways
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t rb = tile / ncb, cb = tile - rb * ncb;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      const int i = COLREAD ? (e & 31) : (e >> 6);
      const int j = COLREAD ? (e >> 5) : (e & 63);
      const int64_t row = row0 + rb * TR + i, col = cb * TC + j;
      t[i * (TC + 1) + j] = (row < n && col < p) ? val(row, col) : 0.0;
    }
    __syncthreads();
    double* dst = K + tile * TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      const int j = e >> 5, i = (e & 31) ^ col_swz(j);  // inverse of in_tile
      dst[e] = t[i * (TC + 1) + j];
    }
    __syncthreads();
  }
}

struct RowMajorSrc {
  const double* src;  // rows [row0, row0 + rows) of an n x p row-major matrix
  int64_t p, row0;
  __device__ double operator()(int64_t r, int64_t c) const { return src[(r - row0) * p + c]; }
};
struct ColMajorSrc {
  const double* src;  // full n x p column-major matrix (device)
  int64_t n;
  __device__ double operator()(int64_t r, int64_t c) const { return src[c * n + r]; }
};
struct GaussSrc {
  uint64_t seed;
  int64_t p_total, col_offset;
  __device__ double operator()(int64_t r, int64_t c) const {
    return det_normal(seed, 0u, (uint64_t)(r * p_total + c + col_offset));
  }
};
struct BlurSrc {
  const double* taps;
  int radius;
  __device__ double operator()(int64_t r, int64_t c) const {
    const int64_t o = r - c;
    return (o >= -radius && o <= radius) ? taps[o + radius] : 0.0;
  }
};

static int fill_grid(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (int)(b > 65535 * 8 ? 65535 * 8 : (b < 1 ? 1 : b));
}
static int tile_grid(int64_t ntiles) { return (int)(ntiles < 148 * 16 ? (ntiles < 1 ? 1 : ntiles) : 148 * 16); }

// rows [row0, row0+rows) of the padded tiled matrix; row0 and rows multiples of TR
void tile_rows_from_rowmajor(double* K, const GemvPlan& pl, const double* src_dev, int64_t row0,
                             int64_t rows, cudaStream_t s) {
  const int64_t ntiles = (rows / TR) * pl.ncb;
  double* dst = K + (row0 / TR) * pl.ncb * TILE;
  fill_tiled_kernel<false><<<tile_grid(ntiles), 256, 0, s>>>(dst, ntiles, pl.ncb, pl.n, pl.p, row0,
                                                              RowMajorSrc{src_dev, pl.p, row0});
  L1G_CUDA(cudaGetLastError());
}

void tile_from_colmajor(double* K, const GemvPlan& pl, const double* src_dev, cudaStream_t s) {
  const int64_t ntiles = pl.nrb * pl.ncb;
  fill_tiled_kernel<true><<<tile_grid(ntiles), 256, 0, s>>>(K, ntiles, pl.ncb, pl.n, pl.p, 0,
                                                             ColMajorSrc{src_dev, pl.n});
  L1G_CUDA(cudaGetLastError());
}

void generate_gaussian(double* K, const GemvPlan& pl, uint64_t seed, int64_t col_offset,
                       int64_t p_total, cudaStream_t s) {
  const int64_t ntiles = pl.nrb * pl.ncb;
  fill_tiled_kernel<true><<<tile_grid(ntiles), 256, 0, s>>>(K, ntiles, pl.ncb, pl.n, pl.p, 0,
                                                             GaussSrc{seed, p_total, col_offset});
  L1G_CUDA(cudaGetLastError());
}

void generate_blur(double* K, const GemvPlan& pl, const double* taps_dev, int radius,
                   cudaStream_t s) {
  const int64_t ntiles = pl.nrb * pl.ncb;
  fill_tiled_kernel<true><<<tile_grid(ntiles), 256, 0, s>>>(K, ntiles, pl.ncb, pl.n, pl.p, 0,
                                                             BlurSrc{taps_dev, radius});
  L1G_CUDA(cudaGetLastError());
}

__global__ void scale_kernel(double* a, int64_t m, double c) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    a[e] = mul(a[e], c);
}
void scale(double* a, int64_t m, double c, cudaStream_t s) {
  scale_kernel<<<fill_grid(m), 256, 0, s>>>(a, m, c);
  L1G_CUDA(cudaGetLastError());
}

// tiled rows [row0, row0+rows) -> row-major (rows x p)
__global__ void untile_kernel(const double* K, double* dst, int64_t ncb, int64_t p,
                              int64_t row0, int64_t rows) {
  const int64_t total = rows * p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / p, c = e - r * p;
    const int64_t row = row0 + r;
    const int64_t rb = row / TR, cb = c / TC;
    dst[e] = K[tile_offset(rb, cb, ncb) + in_tile((int)(row - rb * TR), (int)(c - cb * TC))];
  }
}
void untile_rows(const double* K, const GemvPlan& pl, double* dst, int64_t row0, int64_t rows,
                 cudaStream_t s) {
  untile_kernel<<<fill_grid(rows * pl.p), 256, 0, s>>>(K, dst, pl.ncb, pl.p, row0, rows);
  L1G_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- canonical reductions
// single CTA, 512 threads: pairwise tree over m elements (absent beyond m)
constexpr int RT = 512;
__global__ void __launch_bounds__(RT) reduce_kernel(const double* a, const double* b, int64_t m,
                                                     int op, double* out, int do_sqrt) {
  __shared__ double wv[RT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t ls = 32;
  while (ls < m) ls <<= 1;
  const int64_t nchunks = ls >> 5;
  const int nw = RT / 32;
  const int64_t per = nchunks >= nw ? nchunks / nw : 1;
  const int active = nchunks >= nw ? nw : (int)nchunks;
  auto leaf = [&](int64_t j) -> double {
    if (j >= m) return 0.0;
    const double x = a[j];
    if (op == RED_DOT) return mul(x, b[j]);
    if (op == RED_SQ) return mul(x, x);
    return fabs(x);
  };
  double v = 0.0;
  if (warp < active) {
    if (op == RED_MAX) {
      for (int64_t c = 0; c < per; ++c) v = fmax(v, warp_max(leaf(((int64_t)warp * per + c) * 32 + lane)));
    } else {
      Counter<24> acc;
      for (int64_t c = 0; c < per; ++c)
        acc.push(warp_tree(leaf(((int64_t)warp * per + c) * 32 + lane)), (uint32_t)c);
      v = acc.final_value((uint32_t)per);
    }
  }
  if (lane == 0) wv[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double x = lane < nw ? wv[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < nw; o <<= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, x, o);
      x = op == RED_MAX ? fmax(x, y) : add(x, y);
    }
    if (lane == 0) *out = do_sqrt ? __dsqrt_rn(x) : x;
  }
}
void reduce(const double* a, const double* b, int64_t m, int op, double* out, int do_sqrt,
            cudaStream_t s) {
  reduce_kernel<<<1, RT, 0, s>>>(a, b, m, op, out, do_sqrt);
  L1G_CUDA(cudaGetLastError());
}

__global__ void fill_kernel(double* a, int64_t m, int64_t valid, double c) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    a[e] = e < valid ? c : 0.0;
}
void fill(double* a, int64_t m, int64_t valid, double c, cudaStream_t s) {
  fill_kernel<<<fill_grid(m), 256, 0, s>>>(a, m, valid, c);
  L1G_CUDA(cudaGetLastError());
}

// v = w / *nrm  (linear_operator.cpp:50)
__global__ void div_by_kernel(const double* w, double* v, int64_t m, const double* nrm) {
  const double c = *nrm;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    v[e] = dvd(w[e], c);
}
void div_by(const double* w, double* v, int64_t m, const double* nrm, cudaStream_t s) {
  div_by_kernel<<<fill_grid(m), 256, 0, s>>>(w, v, m, nrm);
  L1G_CUDA(cudaGetLastError());
}

// prox.cpp:23-36
__global__ void soft_threshold_kernel(const double* x, double* out, int64_t m, double t) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[e];
    out[e] = xi > t ? sub(xi, t) : (xi < -t ? add(xi, t) : 0.0);
  }
}
void soft_threshold(const double* x, double* out, int64_t m, double t, cudaStream_t s) {
  soft_threshold_kernel<<<fill_grid(m), 256, 0, s>>>(x, out, m, t);
  L1G_CUDA(cudaGetLastError());
}

// r = kx - y over n elements (Objective misfit for host-side compositions)
__global__ void sub_kernel(const double* a, const double* b, double* out, int64_t m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = sub(a[e], b[e]);
}
void vsub(const double* a, const double* b, double* out, int64_t m, cudaStream_t s) {
  sub_kernel<<<fill_grid(m), 256, 0, s>>>(a, b, out, m);
  L1G_CUDA(cudaGetLastError());
}

// out = a + alpha * b (product rounded, then the sum: Eigen's `a + alpha * b`)
__global__ void lincomb_kernel(const double* a, double alpha, const double* b, double* out,
                               int64_t m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = add(a[e], mul(alpha, b[e]));
}
void lincomb(const double* a, double alpha, const double* b, double* out, int64_t m,
             cudaStream_t s) {
  lincomb_kernel<<<fill_grid(m), 256, 0, s>>>(a, alpha, b, out, m);
  L1G_CUDA(cudaGetLastError());
}

// out = x + coef * (x - xprev)  (FISTA extrapolation, shrinkage.cpp:61-63)
__global__ void extrap_kernel(const double* x, const double* xp, double coef, double* out,
                              int64_t m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = add(x[e], mul(coef, sub(x[e], xp[e])));
}
void extrap(const double* x, const double* xprev, double coef, double* out, int64_t m,
            cudaStream_t s) {
  extrap_kernel<<<fill_grid(m), 256, 0, s>>>(x, xprev, coef, out, m);
  L1G_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- scalar kernels
__global__ void steplength_kernel(l1g_sl_state* sl, const double* dots, l1g_gp_config cfg,
                                  l1g_sl_choice* out) {
  int len = sl->hist_len;
  steplength_from_dots(&sl->tau, sl->hist, &len, dots[0], dots[1], dots[2], cfg, out);
  sl->hist_len = len;
}
void steplength_device(l1g_sl_state* sl, const double* dots, const l1g_gp_config& cfg,
                       l1g_sl_choice* out, cudaStream_t s) {
  steplength_kernel<<<1, 1, 0, s>>>(sl, dots, cfg, out);
  L1G_CUDA(cudaGetLastError());
}

__global__ void backtrack_kernel(const double* in, l1g_gp_config cfg, double* out) {
  double step, f_new;
  int h;
  const bool ok = backtrack_quadratic(in[0], in[1], in[2], in[3], in[4], cfg, &step, &f_new, &h);
  out[0] = step;
  out[1] = f_new;
  out[2] = (double)h;
  out[3] = ok ? 1.0 : 0.0;
}
void backtrack_device(const double* in, const l1g_gp_config& cfg, double* out, cudaStream_t s) {
  backtrack_kernel<<<1, 1, 0, s>>>(in, cfg, out);
  L1G_CUDA(cudaGetLastError());
}

__global__ void state_start_kernel(DevState* st) { st->t_start = globaltimer(); }
void state_start(DevState* st, cudaStream_t s) {
  state_start_kernel<<<1, 1, 0, s>>>(st);
  L1G_CUDA(cudaGetLastError());
}

}  // namespace l1g

namespace l1g {
// harness random streams (bit-identical to orc_normal / orc_uniform)
__global__ void rng_fill_kernel(int kind, uint64_t seed, uint32_t stream, uint64_t first,
                                int64_t count, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = first + (uint64_t)e;
    if (kind == 0) {
      out[e] = det_normal(seed, stream, idx);
    } else {
      uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, 0x5555u};
      philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
      out[e] = u53(c[0], c[1]);
    }
  }
}
void rng_fill(int kind, uint64_t seed, uint32_t stream, uint64_t first, int64_t count,
              double* out, cudaStream_t s) {
  rng_fill_kernel<<<fill_grid(count), 256, 0, s>>>(kind, seed, stream, first, count, out);
  L1G_CUDA(cudaGetLastError());
}
}  // namespace l1g
