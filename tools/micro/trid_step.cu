// Micro-benchmark of the register-tile tridiagonalisation "phase 2" (partial
// row sums of A v over a 4 x 8 register tile + warp-reduced v^T A v + one
// block barrier), 512 threads on one SM.  Variants isolate the pieces.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const double *G, double *out, long long *cyc, int n) {
  __shared__ double vbuf[2][128];
  __shared__ double ps_part[16][128];
  __shared__ double s_red[16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double a[4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[q][u] = G[(32 * q + lane) + 128 * (8 * warp + u)];
  if (tid < 256) vbuf[tid >> 7][tid & 127] = 1.0 / (1 + tid);
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int k = 0; k < n; ++k) {
    const double *vs = vbuf[k & 1];
    double vc[8], vr[4];
#pragma unroll
    for (int u = 0; u < 8; ++u) vc[u] = vs[8 * warp + u];
#pragma unroll
    for (int q = 0; q < 4; ++q) vr[q] = vs[32 * q + lane];
    double vpart = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double s0 = 0, s1 = 0;
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        s0 = fma(a[q][u], vc[u], s0);
        s1 = fma(a[q][u + 1], vc[u + 1], s1);
      }
      const double sacc = s0 + s1;
      if (MODE != 1) ps_part[warp][32 * q + lane] = sacc;
      vpart = fma(vr[q], sacc, vpart);
    }
    if (MODE != 2) vpart = warp_sum(vpart);
    if (lane == 0) s_red[warp] = vpart;
    acc += vpart;
    if (MODE != 3) __syncthreads();
    // a cheap stand-in for the update so the tile stays live and changes
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int u = 0; u < 8; ++u) a[q][u] = fma(-1e-9, vc[u], a[q][u]);
  }
  long long t1 = clock64();
  double r = acc;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int u = 0; u < 8; ++u) r += a[q][u];
  out[tid] = r + ps_part[warp][lane] + s_red[warp];
  if (tid == 0) cyc[0] = t1 - t0;
}
int main() {
  double *G, *o;
  long long *c, h;
  cudaMalloc(&G, 128 * 128 * 8);
  {
    static double hG[128 * 128];
    for (int i = 0; i < 128 * 128; ++i) hG[i] = ((i * 2654435761u) % 1000) * 1e-3 - 0.5;
    cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  }
  cudaMalloc(&o, 512 * 8);
  cudaMalloc(&c, 8);
  const int n = 1000;
  const char *nm[4] = {"full", "no ps_part stores", "no warp_sum", "no barrier"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 512>>>(G, o, c, n);
      if (mode == 1) k<1><<<1, 512>>>(G, o, c, n);
      if (mode == 2) k<2><<<1, 512>>>(G, o, c, n);
      if (mode == 3) k<3><<<1, 512>>>(G, o, c, n);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %.1f cycles / step\n", nm[mode], h / (double)n);
  }
  return 0;
}
