// Fused (s, b) pivots of order n = m + r <= 32, one warp per node
// (P:l.101-106, l.396-399; same outputs as k_pivot_blk / k_pivot_lu_blk).
//
// Waves of many tiny pivots (the 3D and convection-diffusion leaf levels after
// compression, n <= 25) spent their time in a 512-thread CTA per node, one CTA
// per SM at a time.  Here one warp factors one
// pivot, lane i owning rows i + 32 q (q < RPL) of the n x n block in shared
// memory (row stride 32 RPL + 1: conflict-free along rows and columns):
//   SPD: signed Cholesky K = L diag(I_m, -I_r) L^T column by column, then
//        X = L^{-1} by column-oriented forward substitution (lane c = columns
//        c + 32 q);
//   LU:  no-pivot LU, the multiplier growth check (LU_GROWTH_MAX,
//        LORASP_NEED_PIVOT as in k_pivot_lu_blk), L^{-1} (lane c = columns)
//        and U^{-1} (lane c = rows c + 32 q).
// The loops run to n at run time and are not unrolled: a fully unrolled
// 32-column version was bound by instruction fetch (ncu: 62 % of the stall
// samples "no instruction", ~16 k SASS instructions per kernel); restrict-
// qualified row / column pointers let the shared-memory loads run ahead of the
// stores in the inner loops.
#pragma once

namespace lorasp {

template <int RPL>
struct PivW {
  static constexpr int MAXN = 32 * RPL;
  static constexpr int LD = MAXN + 1;
  static constexpr int WARP_DOUBLES = 2 * MAXN * LD + MAXN + 8;   // factor | inverse | 1 / pivots
  static constexpr int WARPS = RPL == 1 ? 2 : 1;                  // nodes per CTA
  static constexpr size_t SMEM = (size_t)WARPS * WARP_DOUBLES * 8;
};
constexpr int PIVW_MAXN = 32;   // (RPL = 2, n <= 64, measured 3x slower than k_pivot_blk: not dispatched)

// dst(i, c) = W[i][c] below the diagonal, on the diagonal 1 (unit) or W[c][c],
// 0 above; lane i stores rows i + 32 q of each column c (coalesced)
template <int RPL>
__device__ __forceinline__ void pivw_store(const double *W, double *dst, int64_t ld, int n, bool unit) {
  constexpr int LD = PivW<RPL>::LD;
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < n; ++c)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i < n) {
        const double v = W[i * LD + c];
        dst[i + (int64_t)c * ld] = (i > c) ? v : (i == c ? (unit ? 1.0 : v) : 0.0);
      }
    }
}

template <int RPL>
__global__ void __launch_bounds__(32 * PivW<RPL>::WARPS) k_pivot_warp(const PivTask *__restrict__ tasks, int ntask,
                                                                      int *status) {
  constexpr int LD = PivW<RPL>::LD, MAXN = PivW<RPL>::MAXN, WARPS = PivW<RPL>::WARPS;
  extern __shared__ double sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int node = blockIdx.x * WARPS + w;
  pdl_trigger();
  if (node >= ntask) return;
  const PivTask t = tasks[node];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  double *S = sh + w * PivW<RPL>::WARP_DOUBLES, *X = S + MAXN * LD, *rdv = X + MAXN * LD;
  for (int c = 0; c < n; ++c)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i < n) S[i * LD + c] = (c <= i) ? t.F[i + (int64_t)c * t.ld] : 0.0;
    }
  __syncwarp();
  // ---- signed Cholesky, d_k = +1 for k < m, -1 after ----
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const double d = (k < t.m) ? 1.0 : -1.0;
    const double v = S[k * LD + k] * d;
    ok = ok && (v > 0.0) && isfinite(v);
    const double rk = frsqrt(fmax(v, 1e-300));
    __syncwarp();
    double lik[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      lik[q] = 0.0;
      if (i == k) {
        S[k * LD + k] = v * rk;
        rdv[k] = rk;
      } else if (i > k && i < n) {
        lik[q] = S[i * LD + k] * (d * rk);
        S[i * LD + k] = lik[q];
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i > k && i < n) {   // distinct rows / columns: restrict lets the loads run ahead of the stores
        const double f = -d * lik[q];
        const double *__restrict__ colk = S + k;
        double *__restrict__ rowi = S + i * LD;
#pragma unroll 4
        for (int jj = k + 1; jj <= i; ++jj) rowi[jj] = fma(f, colk[jj * LD], rowi[jj]);
      }
    }
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0 && atomicCAS(&status[0], 0, -3) == 0) status[1] = t.node;
    return;
  }
  // ---- X = L^{-1}: lane c solves L x = e_c for its columns c + 32 q ----
#pragma unroll
  for (int q = 0; q < RPL; ++q) {
    const int c = lane + 32 * q;
    for (int r = 0; r < n; ++r) X[r * LD + c] = (r == c) ? 1.0 : 0.0;
    if (c < n) {
      double *__restrict__ xc = X + c;
      for (int k = c; k < n; ++k) {
        const double xk = xc[k * LD] * rdv[k];
        xc[k * LD] = xk;
        const double *__restrict__ lk = S + k;
#pragma unroll 4
        for (int r = k + 1; r < n; ++r) xc[r * LD] = fma(-lk[r * LD], xk, xc[r * LD]);
      }
    }
  }
  __syncwarp();
  pivw_store<RPL>(X, t.F, t.ld, n, false);
}

template <int RPL>
__global__ void __launch_bounds__(32 * PivW<RPL>::WARPS) k_pivot_lu_warp(const PivTask *__restrict__ tasks, int ntask,
                                                                         int *status) {
  constexpr int LD = PivW<RPL>::LD, MAXN = PivW<RPL>::MAXN, WARPS = PivW<RPL>::WARPS;
  extern __shared__ double sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int node = blockIdx.x * WARPS + w;
  pdl_trigger();
  if (node >= ntask) return;
  const PivTask t = tasks[node];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  double *S = sh + w * PivW<RPL>::WARP_DOUBLES, *X = S + MAXN * LD, *rdv = X + MAXN * LD;
  double amax = 0.0;
  for (int c = 0; c < n; ++c)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i < n) {
        const double v = t.F[i + (int64_t)c * t.ld];
        S[i * LD + c] = v;
        amax = fmax(amax, fabs(v));
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const double tiny = 1e-14 * amax;
  __syncwarp();
  // ---- no-pivot LU: multipliers below the diagonal, U on and above ----
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const double piv = S[k * LD + k];
    ok = ok && (fabs(piv) > tiny) && isfinite(piv);
    const double rp = frcp(piv);
    if (lane == 0) rdv[k] = rp;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i > k && i < n) {
        double *__restrict__ rowi = S + i * LD;
        const double *__restrict__ rowk = S + k * LD;
        const double lik = rowi[k] * rp;
        rowi[k] = lik;
#pragma unroll 4
        for (int jj = k + 1; jj < n; ++jj) rowi[jj] = fma(-lik, rowk[jj], rowi[jj]);
      }
    }
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0 && atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
    return;
  }
  // multiplier growth (no pivoting), recorded like lu_growth
  double g = 0.0;
#pragma unroll
  for (int q = 0; q < RPL; ++q) {
    const int i = lane + 32 * q;
    for (int c = 0; c < i && i < n; ++c) g = fmax(g, fabs(S[i * LD + c]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
  if (lane == 0) atomicMax(reinterpret_cast<unsigned long long *>(status + 2), (unsigned long long)__double_as_longlong(g));
  if (g > LU_GROWTH_MAX) {
    if (lane == 0 && atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
    return;
  }
  // ---- region 0 <- L^{-1} (unit lower): lane c solves L x = e_c ----
#pragma unroll
  for (int q = 0; q < RPL; ++q) {
    const int c = lane + 32 * q;
    for (int r = 0; r < n; ++r) X[r * LD + c] = (r == c) ? 1.0 : 0.0;
    if (c < n) {
      double *__restrict__ xc = X + c;
      for (int k = c; k < n; ++k) {
        const double xk = xc[k * LD];
        const double *__restrict__ lk = S + k;
#pragma unroll 4
        for (int r = k + 1; r < n; ++r) xc[r * LD] = fma(-lk[r * LD], xk, xc[r * LD]);
      }
    }
  }
  __syncwarp();
  pivw_store<RPL>(X, t.F, t.ld, n, true);
  __syncwarp();
  // ---- region 1 <- U^{-T}: lane c forms rows c + 32 q of U^{-1} (= columns of U^{-T}) ----
#pragma unroll
  for (int q = 0; q < RPL; ++q) {
    const int c = lane + 32 * q;
    for (int r = 0; r < n; ++r) X[r * LD + c] = (r == c) ? 1.0 : 0.0;
    if (c < n) {
      double *__restrict__ yc = X + c;
      for (int j = c; j < n; ++j) {
        const double yj = yc[j * LD] * rdv[j];
        yc[j * LD] = yj;
        const double *__restrict__ uj = S + j * LD;
#pragma unroll 4
        for (int jj = j + 1; jj < n; ++jj) yc[jj * LD] = fma(-yj, uj[jj], yc[jj * LD]);
      }
    }
  }
  __syncwarp();
  double *R1 = t.F2 ? t.F2 : t.F + (int64_t)t.ld * n;
  pivw_store<RPL>(X, R1, t.ld, n, false);
}

}  // namespace lorasp
