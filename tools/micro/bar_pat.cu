// Cost of the "one warp produces, barrier, everyone consumes" step pattern
// (the MGS / Householder skeleton), 512 threads on one SM, cycles per step.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double *out, long long *cyc, int n) {
  __shared__ double buf[2][128];
  __shared__ double red[16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double z[4];
  for (int q = 0; q < 4; ++q) z[q] = 1.0 + 1e-3 * (tid + q);
  if (tid < 256) buf[tid >> 7][tid & 127] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
    double *b = buf[k & 1];
    if (MODE >= 1 && warp == (k & 15)) {          // producer: reduce + publish
      double s = 0;
      for (int q = 0; q < 4; ++q) s = fma(z[q], z[q], s);
      s = warp_sum(s);
      const double inv = (MODE >= 2) ? 1.0 / sqrt(s) : s;
      for (int q = 0; q < 4; ++q) b[32 * q + lane] = z[q] * inv;
    }
    __syncthreads();
    if (MODE >= 3) {                                // consumers: dot + warp_sum + axpy
      double s = 0;
      for (int q = 0; q < 4; ++q) s = fma(b[32 * q + lane], z[q], s);
      s = warp_sum(s);
      for (int q = 0; q < 4; ++q) z[q] = fma(-1e-3 * s, b[32 * q + lane], z[q]);
    }
  }
  long long t1 = clock64();
  out[tid] = z[0] + z[1] + z[2] + z[3];
  if (tid == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o;
  long long *c, h;
  cudaMalloc(&o, 512 * 8);
  cudaMalloc(&c, 8);
  const int n = 2000;
  const char *nm[4] = {"barrier only", "+producer warp_sum/STS", "+sqrt/div", "+consumer dot/axpy"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 512>>>(o, c, n);
      if (mode == 1) k<1><<<1, 512>>>(o, c, n);
      if (mode == 2) k<2><<<1, 512>>>(o, c, n);
      if (mode == 3) k<3><<<1, 512>>>(o, c, n);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-26s %.1f cycles / step\n", nm[mode], h / (double)n);
  }
  return 0;
}
