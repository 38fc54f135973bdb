// lat.cu -- dependent-chain latency of fp64 add/mul/div, floor, int64<->fp64 conversions.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  for (int i = 0; i < 1024; ++i) x = __dmul_rn(x, b);
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) x = __ddiv_rn(x, b);
  long long t3 = clock64();
  for (int i = 0; i < 1024; ++i) x = floor(x * b) + 0.5;
  long long t4 = clock64();
  long long z = (long long)a;
  for (int i = 0; i < 1024; ++i) z = (long long)((double)z * b) + 1;
  long long t5 = clock64();
  double y = a;
  for (int i = 0; i < 1024; ++i) y = (double)((long long)y + 3);
  long long t6 = clock64();
  out[0] = x + z + y;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1.0, 1.0000001);
  k<<<1, 32>>>(o, c, 1.0, 1.0000001);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("DADD %.1f  DMUL %.1f  DDIV %.1f  floor(x*b)+.5 %.1f  ll->d*b->ll+1 %.1f  d->ll+3->d %.1f cycles/iter\n",
         h[0]/1024.0, h[1]/1024.0, h[2]/256.0, h[3]/1024.0, h[4]/1024.0, h[5]/1024.0);
  return 0;
}
