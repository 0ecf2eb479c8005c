// clock64 phase stamps of k_pivot_blk (instrumented copy generated from kernels.cuh)
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "kernels.cuh"
using namespace lorasp;
__global__ void __launch_bounds__(512, 1) k_pivot_prof(const PivTask *__restrict__ tasks, int *status, long long *clk) {
  long long t0 = clock64(); int ns = 0;
  auto stamp = [&]() { if (threadIdx.x == 0 && blockIdx.x == 0 && ns < 60) clk[ns++] = clock64() - t0; };
  // Signed Cholesky K = L D L^T (D = diag(I_m, -I_r)) of the fused pivot with
  // X = L^{-1} built on the fly, one CTA per node, 16-column blocks k:
  //   warp 0 (critical path): trailing update of diagonal block k, its signed
  //     Cholesky in registers (pivb_diag_chol) and W_k = L_kk^{-1}, stored as X_kk;
  //   the other warps, beside it: the rest of the trailing update of step k-1,
  //     and row block k of X (X_kj = -W_k sum_l L_kl X_lj, as M = W_k L_k,: in
  //     place, then -M X into registers, written one phase later);
  //   all warps: the panel L21 = A21 W_k^T D_k.
  // Every product runs on the FP64 tensor cores (m8n8k4 DMMA fragments straight
  // from shared memory); two block barriers per 16 columns.
  extern __shared__ double sh[];
  __shared__ double W[PIVB_NB * PIVB_NB];
  __shared__ double rd[PIVB_MAXN + PIVB_NB];   // 1 / l_kk
  __shared__ double lcol[32];
  __shared__ int s_fail;
  pdl_trigger();
  const PivTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int npad = pivb_npad(n), lda = pivb_lda(n), nb = npad / PIVB_NB;
  const int g = lane >> 2, tq = lane & 3;
  double *A = sh;
  for (int j = warp; j < npad; j += nw)
    for (int i = lane; i < npad; i += 32)
      A[i + j * lda] = (i >= j && i < n && j < n) ? t.F[i + (int64_t)j * t.ld] : 0.0;
  if (tid == 0) s_fail = 0;
  __syncthreads();
  // warp 0: factor diagonal block k (already updated), W = L_kk^{-1}, X_kk = W
  auto diag = [&](int k) {
    const int j0 = PIVB_NB * k, b = min(PIVB_NB, n - j0);
    stamp();
    if (!pivb_diag_chol(A, lda, j0, b, t.m, rd, lane, lcol)) {
      if (lane == 0) {
        s_fail = 1;
        if (atomicCAS(&status[0], 0, -3) == 0) status[1] = t.node;
      }
      return;
    }
    stamp();
    pivb_diag_inverse(A, lda, j0, b, W, lane, rd);
    __syncwarp();
    stamp();
    for (int q = lane; q < PIVB_NB * PIVB_NB; q += 32) {
      const int i = q & 15, c = q >> 4;
      if (i >= c) A[(j0 + i) + (j0 + c) * lda] = W[i + c * PIVB_NB];
    }
  };
  // A22 block (r0, s0) -= L21(r0) D L21(s0)^T over the 16 columns j0..
  auto trail = [&](int j0, int r0, int s0) {
    double c0 = A[(r0 + g) + (s0 + 2 * tq) * lda], c1 = A[(r0 + g) + (s0 + 2 * tq + 1) * lda];
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int kc = j0 + 4 * k4 + tq;
      const double dk = (kc < t.m) ? -1.0 : 1.0;   // -d_k: subtract
      const double av = frag_ld(A, lda, r0, j0 + 4 * k4);
      const double bv = frag_ld(A, lda, s0, j0 + 4 * k4) * dk;
      dmma884(c0, c1, av, bv);
    }
    A[(r0 + g) + (s0 + 2 * tq) * lda] = c0;
    A[(r0 + g) + (s0 + 2 * tq + 1) * lda] = c1;
  };
  if (warp == 0) diag(0);
  __syncthreads();
  if (s_fail) return;
  constexpr int MAXI = 3;   // X items per warp (4 k <= 36 items over 15 warps)
  double xres[MAXI][2];
  int xk = -1;              // row block whose X items are held in xres
  for (int k = 0; k < nb; ++k) {
    const int j0 = PIVB_NB * k, j1 = j0 + PIVB_NB;
    const int nrb = (npad - j1) >> 3;
    // ---- phase B: write X row block k-1; panel L21 of column block k; M = W_k L_k,
    if (xk >= 0 && warp > 0) {
#pragma unroll
      for (int u = 0; u < MAXI; ++u) {
        const int it = (warp - 1) + u * (nw - 1);
        if (it >= 4 * xk) break;
        const int rh = it & 1, cb = it >> 1;
        const int row = PIVB_NB * xk + 8 * rh + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) A[row + (8 * cb + 2 * tq + e) * lda] = xres[u][e];
      }
    }
    for (int it = warp; it < nrb + 2 * k; it += nw) {
      if (it < nrb) {   // panel: L21(8-row block) = A21 (W^T D), B(kk, c) = W[c][kk] d_c
        const int r0 = j1 + 8 * it;
        double af[4];
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) af[k4] = frag_ld(A, lda, r0, j0 + 4 * k4);
        double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          const int col = 8 * cb + g;
          const double dc = (j0 + col < t.m) ? 1.0 : -1.0;
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) dmma884(c[cb][0], c[cb][1], af[k4], W[col + (4 * k4 + tq) * PIVB_NB] * dc);
        }
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < 2; ++cb)
#pragma unroll
          for (int e = 0; e < 2; ++e) A[(r0 + g) + (j0 + 8 * cb + 2 * tq + e) * lda] = c[cb][e];
      } else {          // M(:, 8-col block cb) = W L_k(:, cb), both row halves, in place
        const int cb = it - nrb;
        double bf[4];
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) bf[k4] = A[(j0 + 4 * k4 + tq) + (8 * cb + g) * lda];
        double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int rh = 0; rh < 2; ++rh)
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) dmma884(c[rh][0], c[rh][1], W[(8 * rh + g) + (4 * k4 + tq) * PIVB_NB], bf[k4]);
        __syncwarp();
#pragma unroll
        for (int rh = 0; rh < 2; ++rh)
#pragma unroll
          for (int e = 0; e < 2; ++e) A[(j0 + 8 * rh + g) + (8 * cb + 2 * tq + e) * lda] = c[rh][e];
      }
    }
    __syncthreads();
    // ---- phase C: warp 0 updates + factors diagonal block k+1; the others: the
    // rest of the trailing update and X row block k = -M X (registers)
    if (warp == 0) {
      if (nrb > 0) {
        trail(j0, j1, j1);
        trail(j0, j1 + 8, j1);
        trail(j0, j1 + 8, j1 + 8);
        __syncwarp();
        diag(k + 1);
      }
    } else {
      const int npair = nrb * (nrb + 1) / 2;
      for (int q = warp - 1 + 3; q < npair; q += nw - 1) {   // pairs 0..2 = diagonal block k+1
        int ib = (int)((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
        while ((ib + 1) * (ib + 2) / 2 <= q) ++ib;
        while (ib * (ib + 1) / 2 > q) --ib;
        const int jb = q - ib * (ib + 1) / 2;
        trail(j0, j1 + 8 * ib, j1 + 8 * jb);
      }
#pragma unroll
      for (int u = 0; u < MAXI; ++u) {
        const int it = (warp - 1) + u * (nw - 1);
        if (it >= 4 * k) break;
        const int rh = it & 1, cb = it >> 1;
        const int r0 = j0 + 8 * rh;
        double c0 = 0.0, c1 = 0.0;
        for (int k0 = 8 * cb; k0 < j0; k0 += 4) {   // X(l, col) = 0 for l < col
          const double av = A[(r0 + g) + (k0 + tq) * lda];           // M(row, l)
          double bv = A[(k0 + tq) + (8 * cb + g) * lda];             // X(l, col)
          if (k0 + tq < 8 * cb + g) bv = 0.0;
          dmma884(c0, c1, av, bv);
        }
        xres[u][0] = -c0;
        xres[u][1] = -c1;
      }
      xk = k;
    }
    __syncthreads();
    if (s_fail) return;
  }
  if (warp > 0 && xk >= 0) {   // the last X row block
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int it = (warp - 1) + u * (nw - 1);
      if (it >= 4 * xk) break;
      const int rh = it & 1, cb = it >> 1;
      const int row = PIVB_NB * xk + 8 * rh + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) A[row + (8 * cb + 2 * tq + e) * lda] = xres[u][e];
    }
  }
  __syncthreads();
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i < n; i += 32) t.F[i + (int64_t)j * t.ld] = (i >= j) ? A[i + j * lda] : 0.0;
  __syncthreads();
  stamp();
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[63] = ns;
}

int main() {
  cudaFuncSetAttribute(k_pivot_prof, cudaFuncAttributeMaxDynamicSharedMemorySize, 215 * 1024);
  int ns[] = {32, 64, 128};
  double *K; int *st; PivTask *dt; long long *clk;
  cudaMalloc(&K, 160 * 160 * 8 * 2); cudaMalloc(&st, 64); cudaMalloc(&dt, sizeof(PivTask)); cudaMalloc(&clk, 64 * 8);
  for (int q = 0; q < 3; ++q) {
    const int n = ns[q], r = n / 4, m = n - r;
    std::vector<double> h((size_t)n * n, 0.0);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double v = (i == j) ? (i < m ? 4.0 : 0.0) : ((i < m && j < m && (i - j == 1 || j - i == 1)) ? -1.0 : 0.0);
        if (i >= m && j < m && (i - m) == (j % r)) v = 0.3;
        if (j >= m && i < m && (j - m) == (i % r)) v = 0.3;
        h[i + (size_t)j * n] = v;
      }
    PivTask t{}; t.F = K; t.ld = n; t.m = m; t.r = r;
    cudaMemcpy(dt, &t, sizeof(t), cudaMemcpyHostToDevice);
    long long hc[64];
    for (int it = 0; it < 3; ++it) {
      cudaMemcpy(K, h.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
      cudaMemset(st, 0, 64);
      k_pivot_prof<<<1, 512, pivb_smem_bytes(n)>>>(dt, st, clk);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(hc, clk, 64 * 8, cudaMemcpyDeviceToHost);
    printf("n=%d stamps:", n);
    for (int s = 0; s < hc[63]; ++s) printf(" %lld", hc[s]);
    printf("\n");
  }
  return 0;
}
