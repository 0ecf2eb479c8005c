#include <cstdio>
#include <cuda_runtime.h>
#include "kernels.cuh"
using namespace lorasp;
namespace lorasp {
__device__ __forceinline__ bool lu_dbg(double *__restrict__ A, int lda, int j0, int b, double tiny,
                                               double *__restrict__ rd, int lane, double *urow) {
  // Branch-free (selects only): the pivot row reaches the other lanes through
  // shared memory (urow, >= 16 doubles) instead of one shuffle per column entry;
  // a vanishing pivot is accumulated in the result, not a break.
  const int i = lane;
  double a[PIVB_NB];
#pragma unroll
  for (int c = 0; c < PIVB_NB; ++c) a[c] = (i < b && c < b) ? A[(j0 + i) + (j0 + c) * lda] : 0.0;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < PIVB_NB; ++k) {
    if (k < b) {
      if (i == k) {
#pragma unroll
        for (int jj = k; jj < PIVB_NB; ++jj) urow[jj] = a[jj];
      }
      __syncwarp();
      const double piv = urow[k];
      ok = ok && (fabs(piv) > tiny) && isfinite(piv);
      if (k < 3 && i < 3) printf("k=%d lane=%d piv=%g a=%g ok=%d\n", k, i, piv, a[k], (int)ok);
      const double rp = frcp(piv);
      rd[j0 + k] = rp;   // every lane stores the same value
      const double lik = a[k] * rp;
      a[k] = (i > k) ? lik : a[k];
#pragma unroll
      for (int jj = k + 1; jj < PIVB_NB; ++jj) {
        const double u = fma(-lik, urow[jj], a[jj]);
        a[jj] = (jj < b && i > k) ? u : a[jj];
      }
      __syncwarp();
    }
  }
  if (ok) {
#pragma unroll
    for (int c = 0; c < PIVB_NB; ++c)
      if (i < b && c < b) A[(j0 + i) + (j0 + c) * lda] = a[c];
  }
  __syncwarp();
  return ok;
}

}

__global__ void k(double *out, int *okout) {
  __shared__ double A[16 * 17], rd[32], urow[16];
  const int lane = threadIdx.x;
  for (int q = lane; q < 16 * 17; q += 32) {
    const int i = q % 17, j = q / 17;
    A[q] = (i == j) ? 4.0 : ((i < 16 && (i - j == 1 || j - i == 1)) ? -1.0 : 0.0);
  }
  __syncwarp();
  bool ok = lu_dbg(A, 17, 0, 16, 1e-14 * 4, rd, lane, urow);
  if (lane == 0) okout[0] = ok;
  for (int q = lane; q < 16 * 17; q += 32) out[q] = A[q];
  if (lane < 16) out[300 + lane] = rd[lane];
}
int main() {
  double *o; int *ok; cudaMalloc(&o, 400 * 8); cudaMalloc(&ok, 4);
  k<<<1, 32>>>(o, ok);
  double h[400]; int hk;
  cudaMemcpy(h, o, 400 * 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hk, ok, 4, cudaMemcpyDeviceToHost);
  printf("ok=%d  u00=%g u11=%g l10=%g l21=%g rd0=%g rd1=%g err=%s\n", hk, h[0], h[1 + 17], h[1], h[2 + 17], h[300], h[301],
         cudaGetErrorString(cudaGetLastError()));
}
