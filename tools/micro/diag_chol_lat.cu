// Cycles of the fused-pivot diagonal-block chain (pivb_diag_chol: 16-column
// signed Cholesky by one warp, lane = row) and of two restructured variants.
#include <cstdio>
#include <cuda_runtime.h>
#include "kernels.cuh"
using namespace lorasp;

// variant: no early exit (failure flag accumulated), row broadcast of each column's
// multipliers through shared memory instead of 15 shuffles per column
__device__ __forceinline__ bool diag_chol_v2(double *__restrict__ A, int lda, int j0, int b, int m,
                                             double *__restrict__ rd, int lane, double *__restrict__ lcol) {
  const int i = lane;
  double a[PIVB_NB];
#pragma unroll
  for (int c = 0; c < PIVB_NB; ++c) a[c] = (i < b && c <= i) ? A[(j0 + i) + (j0 + c) * lda] : 0.0;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < PIVB_NB; ++k) {
    if (k < b) {
      const double d = (j0 + k < m) ? 1.0 : -1.0;
      const double v = __shfl_sync(0xffffffffu, a[k], k) * d;
      ok = ok && (v > 0.0);
      const double rk = frsqrt(fmax(v, 1e-300));
      const double lik = (i > k) ? a[k] * (d * rk) : 0.0;
      if (i == k) a[k] = v * rk;
      else if (i > k) a[k] = lik;
      if (lane == 0) rd[j0 + k] = rk;
      if (i < PIVB_NB) lcol[i] = lik;
      __syncwarp();
      const double f = -d * lik;
#pragma unroll
      for (int jj = k + 1; jj < PIVB_NB; ++jj)
        if (jj < b && i >= jj) a[jj] = fma(f, lcol[jj], a[jj]);
      __syncwarp();
    }
  }
#pragma unroll
  for (int c = 0; c < PIVB_NB; ++c)
    if (i < b && c <= i) A[(j0 + i) + (j0 + c) * lda] = a[c];
  __syncwarp();
  return ok;
}

// v3: column k of L parked in its own 16-slot row of smem (one warp barrier per
// column, no reuse hazard), no early exit, the next column's update first
__device__ __forceinline__ bool diag_chol_v3(double *__restrict__ A, int lda, int j0, int b, int m,
                                             double *__restrict__ rd, int lane, double *__restrict__ lc) {
  const int i = lane;
  double a[PIVB_NB];
#pragma unroll
  for (int c = 0; c < PIVB_NB; ++c) a[c] = (i < b && c <= i) ? A[(j0 + i) + (j0 + c) * lda] : 0.0;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < PIVB_NB; ++k) {
    if (k < b) {
      const double d = (j0 + k < m) ? 1.0 : -1.0;
      const double v = __shfl_sync(0xffffffffu, a[k], k) * d;
      ok = ok && (v > 0.0);
      const double rk = frsqrt(fmax(v, 1e-300));
      const double lik = (i > k) ? a[k] * (d * rk) : 0.0;
      if (i == k) a[k] = v * rk;
      else if (i > k) a[k] = lik;
      if (i < PIVB_NB) lc[k * PIVB_NB + i] = lik;
      if (lane == 0) rd[j0 + k] = rk;
      __syncwarp();
      const double f = -d * lik;
#pragma unroll
      for (int jj = k + 1; jj < PIVB_NB; ++jj)
        if (jj < b && i >= jj) a[jj] = fma(f, lc[k * PIVB_NB + jj], a[jj]);
    }
  }
#pragma unroll
  for (int c = 0; c < PIVB_NB; ++c)
    if (i < b && c <= i) A[(j0 + i) + (j0 + c) * lda] = a[c];
  __syncwarp();
  return ok;
}

template <int V>
__global__ void k_bench(double *g, long long *out, int reps) {
  __shared__ double A[16 * 17], rd[32], lcol[32], W[256], lc[256];
  const int lane = threadIdx.x;
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    for (int q = lane; q < 16 * 17; q += 32) {
      const int i = q % 17, j = q / 17;
      A[q] = (i == j) ? 4.0 : ((i < 16 && (i - j == 1 || j - i == 1)) ? -1.0 : 0.0);
    }
    __syncwarp();
    const long long t0 = clock64();
    bool ok;
    if (V == 0 || V == 2) ok = pivb_diag_chol(A, 17, 0, 16, 16, rd, lane, lcol);
    else if (V == 1) ok = diag_chol_v2(A, 17, 0, 16, 16, rd, lane, lcol);
    else ok = diag_chol_v3(A, 17, 0, 16, 16, rd, lane, lc);
    const long long t1 = clock64();
    if (V == 2) pivb_diag_inverse(A, 17, 0, 16, W, lane, rd);
    const long long t2 = clock64();
    if (!ok) g[0] = 1.0;
    best = min(best, V == 2 ? t2 - t1 : t1 - t0);
  }
  if (lane == 0) out[V] = best;
  if (lane == 0) g[1] = A[5] + W[3];
}

// the same chain inside a 512-thread block under `if (warp == 0)` (the k_pivot_blk context)
template <int V>
__global__ void __launch_bounds__(512, 1) k_bench512(double *g, long long *out, int reps) {
  __shared__ double A[16 * 17], rd[32], lcol[32], W[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    for (int q = threadIdx.x; q < 16 * 17; q += blockDim.x) {
      const int i = q % 17, j = q / 17;
      A[q] = (i == j) ? 4.0 : ((i < 16 && (i - j == 1 || j - i == 1)) ? -1.0 : 0.0);
    }
    __syncthreads();
    if (V == 0 ? warp == 0 : __shfl_sync(0xffffffffu, warp, 0) == 0) {
      const long long t0 = clock64();
      const bool ok = pivb_diag_chol(A, 17, 0, 16, 16, rd, lane, lcol);
      const long long t1 = clock64();
      if (!ok) g[0] = 1.0;
      best = min(best, t1 - t0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[4 + V] = best;
}

int main() {
  double *g; long long *o, h[4];
  cudaMalloc(&g, 64); cudaMalloc(&o, 64);
  k_bench<0><<<1, 32>>>(g, o, 20);
  k_bench<1><<<1, 32>>>(g, o, 20);
  k_bench<2><<<1, 32>>>(g, o, 20);
  k_bench<3><<<1, 32>>>(g, o, 20);
  k_bench512<0><<<1, 512>>>(g, o, 20);
  k_bench512<1><<<1, 512>>>(g, o, 20);
  long long h2[2];
  cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, o + 4, 16, cudaMemcpyDeviceToHost);
  printf("{\"in_512_block_if_warp0\": %lld, \"in_512_block_shfl_uniform\": %lld}\n", h2[0], h2[1]);
  printf("{\"diag_chol_cycles\": %lld, \"diag_chol_v2_cycles\": %lld, \"diag_inverse_cycles\": %lld, \"diag_chol_v3_cycles\": %lld}\n", h[0], h[1], h[2], h[3]);
  return 0;
}
