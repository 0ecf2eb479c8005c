// FP64 throughput / block-synchronisation micro-benchmarks on one SM (cycles).
//   dfma_tp : 512 threads x 8 independent DFMA chains -> DFMA per clock per SM
//   bar     : __syncthreads() round trip with 16 warps (nothing else)
//   wsum    : warp_sum of a double (5 xor-shuffle rounds), dependent chain
//   lds     : dependent shared-memory load chain (pointer chasing)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
  __shared__ int chase[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) chase[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = a + j;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], b, a);
  __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t2 = clock64();
  double s = x[0];
  for (int i = 0; i < n; ++i)
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  long long t3 = clock64();
  int p = threadIdx.x & 1023;
  for (int i = 0; i < n; ++i) p = chase[p];
  long long t4 = clock64();
  double r = s + p;
  for (int j = 0; j < 8; ++j) r += x[j];
  out[threadIdx.x] = r;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double *o; long long *c, h[4]; cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
  int n = 2048;
  for (int it = 0; it < 2; ++it) k<<<1, 512>>>(o, c, 0.5, 0.999, n);
  cudaDeviceSynchronize();
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("dfma/clk/SM %.1f  bar(16 warps) %.1f cyc  warp_sum(double) %.1f cyc  lds chain %.1f cyc\n",
         512.0 * 8 * n / h[0], h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
  return 0;
}
