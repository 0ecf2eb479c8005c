// Fused (s, b) pivots of order n = m + r <= 32, one warp per node
// (P:l.101-106, l.396-399; same outputs as k_pivot_blk / k_pivot_lu_blk).
//
// Waves of many tiny pivots (the 3D and convection-diffusion leaf levels after
// compression, n <= 25) spent their time in a 512-thread CTA per node, one CTA
// per SM at a time.  Here one warp factors one pivot, lane i owning row i of
// the n x n block in shared memory (row stride 33: conflict-free both ways):
//   SPD: signed Cholesky K = L diag(I_m, -I_r) L^T column by column, then
//        X = L^{-1} by column-oriented forward substitution (lane c = column c);
//   LU:  no-pivot LU, the multiplier growth check (LU_GROWTH_MAX,
//        LORASP_NEED_PIVOT as in k_pivot_lu_blk), L^{-1} (lane c = column c)
//        and U^{-1} (lane c = row c).
// The loops run to n at run time and are not unrolled: a fully unrolled
// 32-column version was bound by instruction fetch (ncu: 62 % of the stall
// samples "no instruction", ~16 k SASS instructions per kernel).
#pragma once

namespace lorasp {

constexpr int PIVW_MAXN = 32;
constexpr int PIVW_LD = 33;                                   // row stride
constexpr int PIVW_WARP_DOUBLES = 2 * 32 * PIVW_LD + 32 + 8;  // factor | inverse | 1 / pivots
constexpr int PIVW_WARPS = 2;                                  // nodes per CTA

// dst(i, c) = W[i][c] below the diagonal (W: row stride PIVW_LD), diag on the
// diagonal (1 for a unit factor, else W[c][c]), 0 above; lane i stores row i of
// each column c (coalesced)
__device__ __forceinline__ void pivw_store(const double *W, double *dst, int64_t ld, int n, bool unit) {
  const int i = threadIdx.x & 31;
  if (i >= n) return;
  for (int c = 0; c < n; ++c) {
    const double v = W[i * PIVW_LD + c];
    dst[i + (int64_t)c * ld] = (i > c) ? v : (i == c ? (unit ? 1.0 : v) : 0.0);
  }
}

__global__ void __launch_bounds__(32 * PIVW_WARPS) k_pivot_warp(const PivTask *__restrict__ tasks, int ntask,
                                                                int *status) {
  __shared__ double sh[PIVW_WARPS * PIVW_WARP_DOUBLES];
  const int w = threadIdx.x >> 5, i = threadIdx.x & 31;
  const int node = blockIdx.x * PIVW_WARPS + w;
  pdl_trigger();
  if (node >= ntask) return;
  const PivTask t = tasks[node];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  double *S = sh + w * PIVW_WARP_DOUBLES, *X = S + 32 * PIVW_LD, *rdv = X + 32 * PIVW_LD;
  for (int c = 0; c < n; ++c)
    if (i < n) S[i * PIVW_LD + c] = (c <= i) ? t.F[i + (int64_t)c * t.ld] : 0.0;
  __syncwarp();
  // ---- signed Cholesky, d_k = +1 for k < m, -1 after ----
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const double d = (k < t.m) ? 1.0 : -1.0;
    const double v = S[k * PIVW_LD + k] * d;
    ok = ok && (v > 0.0) && isfinite(v);
    const double rk = frsqrt(fmax(v, 1e-300));
    __syncwarp();
    double lik = 0.0;
    if (i == k) {
      S[k * PIVW_LD + k] = v * rk;
      rdv[k] = rk;
    } else if (i > k && i < n) {
      lik = S[i * PIVW_LD + k] * (d * rk);
      S[i * PIVW_LD + k] = lik;
    }
    __syncwarp();
    if (i > k && i < n) {   // distinct rows / columns: restrict lets the loads run ahead of the stores
      const double f = -d * lik;
      const double *__restrict__ colk = S + k;
      double *__restrict__ rowi = S + i * PIVW_LD;
#pragma unroll 4
      for (int jj = k + 1; jj <= i; ++jj) rowi[jj] = fma(f, colk[jj * PIVW_LD], rowi[jj]);
    }
    __syncwarp();
  }
  if (!ok) {
    if (i == 0 && atomicCAS(&status[0], 0, -3) == 0) status[1] = t.node;
    return;
  }
  // ---- X = L^{-1}: lane c solves L x = e_c, x in column c of X ----
  for (int q = 0; q < n; ++q) X[q * PIVW_LD + i] = (q == i) ? 1.0 : 0.0;
  if (i < n) {
    double *__restrict__ xc = X + i;
    for (int k = i; k < n; ++k) {
      const double xk = xc[k * PIVW_LD] * rdv[k];
      xc[k * PIVW_LD] = xk;
      const double *__restrict__ lk = S + k;
#pragma unroll 4
      for (int q = k + 1; q < n; ++q) xc[q * PIVW_LD] = fma(-lk[q * PIVW_LD], xk, xc[q * PIVW_LD]);
    }
  }
  __syncwarp();
  pivw_store(X, t.F, t.ld, n, false);
}

__global__ void __launch_bounds__(32 * PIVW_WARPS) k_pivot_lu_warp(const PivTask *__restrict__ tasks, int ntask,
                                                                   int *status) {
  __shared__ double sh[PIVW_WARPS * PIVW_WARP_DOUBLES];
  const int w = threadIdx.x >> 5, i = threadIdx.x & 31;
  const int node = blockIdx.x * PIVW_WARPS + w;
  pdl_trigger();
  if (node >= ntask) return;
  const PivTask t = tasks[node];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  double *S = sh + w * PIVW_WARP_DOUBLES, *X = S + 32 * PIVW_LD, *rdv = X + 32 * PIVW_LD;
  double amax = 0.0;
  for (int c = 0; c < n; ++c)
    if (i < n) {
      const double v = t.F[i + (int64_t)c * t.ld];
      S[i * PIVW_LD + c] = v;
      amax = fmax(amax, fabs(v));
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const double tiny = 1e-14 * amax;
  __syncwarp();
  // ---- no-pivot LU: multipliers below the diagonal, U on and above ----
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const double piv = S[k * PIVW_LD + k];
    ok = ok && (fabs(piv) > tiny) && isfinite(piv);
    const double rp = frcp(piv);
    if (i == 0) rdv[k] = rp;
    if (i > k && i < n) {
      double *__restrict__ rowi = S + i * PIVW_LD;
      const double *__restrict__ rowk = S + k * PIVW_LD;
      const double lik = rowi[k] * rp;
      rowi[k] = lik;
#pragma unroll 4
      for (int jj = k + 1; jj < n; ++jj) rowi[jj] = fma(-lik, rowk[jj], rowi[jj]);
    }
    __syncwarp();
  }
  if (!ok) {
    if (i == 0 && atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
    return;
  }
  // multiplier growth (no pivoting), recorded like lu_growth
  double g = 0.0;
  for (int c = 0; c < i && i < n; ++c) g = fmax(g, fabs(S[i * PIVW_LD + c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
  if (i == 0) atomicMax(reinterpret_cast<unsigned long long *>(status + 2), (unsigned long long)__double_as_longlong(g));
  if (g > LU_GROWTH_MAX) {
    if (i == 0 && atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
    return;
  }
  // ---- region 0 <- L^{-1} (unit lower): lane c solves L x = e_c ----
  for (int q = 0; q < n; ++q) X[q * PIVW_LD + i] = (q == i) ? 1.0 : 0.0;
  if (i < n) {
    double *__restrict__ xc = X + i;
    for (int k = i; k < n; ++k) {
      const double xk = xc[k * PIVW_LD];
      const double *__restrict__ lk = S + k;
#pragma unroll 4
      for (int q = k + 1; q < n; ++q) xc[q * PIVW_LD] = fma(-lk[q * PIVW_LD], xk, xc[q * PIVW_LD]);
    }
  }
  __syncwarp();
  pivw_store(X, t.F, t.ld, n, true);
  __syncwarp();
  // ---- region 1 <- U^{-T}: lane c forms row c of U^{-1} (= column c of U^{-T}) ----
  for (int q = 0; q < n; ++q) X[q * PIVW_LD + i] = (q == i) ? 1.0 : 0.0;
  if (i < n) {
    double *__restrict__ yc = X + i;
    for (int j = i; j < n; ++j) {
      const double yj = yc[j * PIVW_LD] * rdv[j];
      yc[j * PIVW_LD] = yj;
      const double *__restrict__ uj = S + j * PIVW_LD;
#pragma unroll 4
      for (int jj = j + 1; jj < n; ++jj) yc[jj * PIVW_LD] = fma(-yj, uj[jj], yc[jj * PIVW_LD]);
    }
  }
  __syncwarp();
  double *R1 = t.F2 ? t.F2 : t.F + (int64_t)t.ld * n;
  pivw_store(X, R1, t.ld, n, false);
}

}  // namespace lorasp
