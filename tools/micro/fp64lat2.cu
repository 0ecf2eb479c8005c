#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ double my_rcp(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r);
  e = fma(-x, r, 1.0); r = fma(r, e, r);
  return r;
}
__device__ __forceinline__ double my_rsqrt(double x) {
  double r; asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(x));
  double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}
__device__ __forceinline__ double my_sqrt(double x) {
  double r = my_rsqrt(x); double s = x * r;
  return x == 0.0 ? 0.0 : fma(0.5 * r, fma(-s, s, x), s);
}
__global__ void k(double *out, long long *cyc, double a, double b, int n, double *acc) {
  double x = a, y = b, z = a, w = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = my_rcp(x + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = sqrt(y + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) z = my_sqrt(z + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) w = __drcp_rn(w + 1.0);
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + w;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  // accuracy over a range
  double maxr = 0, maxs = 0;
  for (int i = 1; i < 20000; ++i) {
    double v = (1.0 + 0.37 * i) * pow(10.0, (double)((i % 61) - 30));
    double r1 = my_rcp(v), r2 = 1.0 / v;
    maxr = fmax(maxr, fabs(r1 - r2) / fabs(r2));
    double s1 = my_sqrt(v), s2 = sqrt(v);
    maxs = fmax(maxs, fabs(s1 - s2) / s2);
  }
  if (threadIdx.x == 0) { acc[0] = maxr; acc[1] = maxs; }
}
int main() {
  double *o, *acc, ha[2]; long long *c, h[4]; cudaMalloc(&o, 1024); cudaMalloc(&c, 64); cudaMalloc(&acc, 16);
  int n = 4096;
  k<<<1, 32>>>(o, c, 0.5, 0.999, n, acc); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 0.5, 0.999, n, acc); cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost); cudaMemcpy(ha, acc, 16, cudaMemcpyDeviceToHost);
  printf("cycles/op: my_rcp+add %.1f  sqrt+add %.1f  my_sqrt+add %.1f  drcp_rn+add %.1f ; max rel err my_rcp %.2e my_sqrt %.2e\n",
         h[0]/(double)n, h[1]/(double)n, h[2]/(double)n, h[3]/(double)n, ha[0], ha[1]);
  return 0;
}
