// fp64_peak.cu -- FP64 throughput on this GPU: DFMA, separate DMUL+DADD, and DMMA (mma.sync
// m8n8k4 f64), each with independent chains.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
constexpr int IT = 4096;
__global__ void k_fma(double* out, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __fma_rn(x[i], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_muladd(double* out, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dmma(double* out, double a, double b) {
  double c[4][2];
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x;
  double A = a + threadIdx.x, B = b;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(A), "d"(B));
  double s = 0;
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256;
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) k_fma<<<blocks, threads>>>(o, 1.0000001, 1e-9);
      if (k == 1) k_muladd<<<blocks, threads>>>(o, 1.0000001, 1e-9);
      if (k == 2) k_dmma<<<blocks, threads>>>(o, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops;
    if (k < 2) flops = 2.0 * 8 * IT * (double)blocks * threads;
    else flops = 2.0 * 8 * 8 * 4 * 4 * IT * (double)blocks * threads / 32;  // per warp mma: 512 flop
    printf("%s: %.3f ms, %.1f TFLOP/s\n", k == 0 ? "DFMA" : (k == 1 ? "DMUL+DADD" : "DMMA m8n8k4"), ms,
           flops / ms / 1e9);
  }
  return 0;
}
