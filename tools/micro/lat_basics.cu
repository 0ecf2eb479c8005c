// Basic latencies on one SM (cycles per iteration, clock64): DFMA chain, warp
// double sum (5 xor stages), __syncthreads (256 / 512 threads), shared store ->
// syncwarp -> load round trip, frsqrt-style chain, a 32-term dot from shared
// memory, and the DFMA chain with W warps running it at once.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double frsqrt(double x) {
  double r = rsqrt(x);   // MUFU.RSQ64H + refinement by the compiler? use explicit Newton
  return r;
}
template <int T>
__global__ void k(double *out, long long *cyc, double a, int n) {
  __shared__ double sh[2048];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 2048; i += blockDim.x) sh[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  double x = a + tid * 1e-9, y = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (T == 0) x = fma(x, 0.999, a);
    if (T == 1) x = warp_sum(x) * 1e-3;
    if (T == 2) { __syncthreads(); x += 1.0; }
    if (T == 3) { sh[lane] = x; __syncwarp(); x = sh[(lane + 1) & 31] * 0.5; __syncwarp(); }
    if (T == 4) x = rsqrt(x) + 0.5;
    if (T == 5) {
      double s0 = 0, s1 = 0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) { s0 = fma(sh[j] , x, s0); s1 = fma(sh[j + 1], x, s1); }
      x = (s0 + s1) * 1e-3;
    }
    if (T == 6) { x = x * 0.5 + 1.0; double q = __dsqrt_rn(x); x = q; }
    if (T == 7) { x = 1.0 / (x + 3.0); }
    if (T == 8) { sh[tid] = x; __syncthreads(); x = sh[(tid + 33) % blockDim.x] * 0.5 + 0.25; __syncthreads(); }
  }
  long long t1 = clock64();
  out[tid] = x + y;
  if (tid == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o;
  long long *c, h;
  cudaMalloc(&o, 1024 * 8);
  cudaMalloc(&c, 8);
  const int n = 2000;
  const char *nm[] = {"dfma chain", "warp_sum f64", "syncthreads", "sts-syncwarp-lds", "rsqrt()", "dot32 from smem",
                      "dsqrt_rn", "ddiv", "sts-bar-lds-bar"};
  int thr[] = {32, 256, 512};
  for (int t : thr) {
    for (int T = 0; T < 9; ++T) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (T) {
          case 0: k<0><<<1, t>>>(o, c, 1.0, n); break;
          case 1: k<1><<<1, t>>>(o, c, 1.0, n); break;
          case 2: k<2><<<1, t>>>(o, c, 1.0, n); break;
          case 3: k<3><<<1, t>>>(o, c, 1.0, n); break;
          case 4: k<4><<<1, t>>>(o, c, 1.0, n); break;
          case 5: k<5><<<1, t>>>(o, c, 1.0, n); break;
          case 6: k<6><<<1, t>>>(o, c, 1.0, n); break;
          case 7: k<7><<<1, t>>>(o, c, 1.0, n); break;
          case 8: k<8><<<1, t>>>(o, c, 1.0, n); break;
        }
      }
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("threads %3d  %-18s %7.1f cycles\n", t, nm[T], h / (double)n);
    }
  }
  return 0;
}
