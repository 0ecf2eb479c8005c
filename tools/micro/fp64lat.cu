// FP64 dependent-chain latency micro-benchmark (cycles per op), one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);            // DFMA chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = y / (x + 2.0);           // DIV chain (+DADD)
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) { z = fma(z, b, a); if (fabs(z) > 1e100) z *= 1e-100; }  // chain w/ compare+select
  long long t3 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) w = w + b;                   // DADD chain
  long long t4 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = fmaf(f, (float)b, (float)a);
  long long t5 = clock64();
  out[threadIdx.x] = x + y + z + w + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double *o; long long *c, h[5]; cudaMalloc(&o, 1024); cudaMalloc(&c, 64);
  int n = 4096;
  k<<<1, 32>>>(o, c, 0.5, 0.999, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 0.5, 0.999, n); cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("cycles/op: dfma %.1f  ddiv+dadd %.1f  dfma+cmp+sel %.1f  dadd %.1f  ffma %.1f\n",
         h[0]/(double)n, h[1]/(double)n, h[2]/(double)n, h[3]/(double)n, h[4]/(double)n);
  return 0;
}
