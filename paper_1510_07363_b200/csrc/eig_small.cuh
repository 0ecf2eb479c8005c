// Compress eigen-solver for small stacks (m <= 64), one CTA per node.
//
// Same algorithm and outputs as the k_tridiag_reg + k_eig_t pair (Householder
// tridiagonalisation of the Gram matrix G = M^T M, Sturm multisection for the
// eigenvalues, rank by Eq. cutOff1 / curOff6, inverse iteration, MGS,
// back-transformation; P:l.319-359, l.580-584), fused into one launch and laid
// out for latency, since the upper levels' waves hold few nodes and every step
// of the tridiagonalisation is a dependent chain:
//   * G lives in registers (QR row groups x 8 columns per thread, 4 QR warps);
//   * two block barriers per Householder step instead of three: after the
//     partial products A v every warp forms the whole p = tau A v for its rows
//     and the reduction p.v itself (the same values in the same order, so every
//     warp holds bitwise the same w = p + alpha v), the column entries of w
//     arrive by shuffles;
//   * the warp owning column k+1 forms v_{k+1} straight after its own update;
//   * the reflectors stay in shared memory for the back-transformation.
// Dynamic shared memory: eig_small_smem_bytes(QR).
#pragma once

namespace lorasp {

__host__ __device__ constexpr int eig_small_smem_doubles(int QR) {
  return (32 * QR) * (32 * QR)            /* reflectors, v_j at [j m] */
         + 5 * (32 * QR + 8)              /* d, e, tau, e2 (padded), lam */
         + 2 * 32 * QR                    /* MGS broadcast buffer */
         + 5 * (32 * QR) * (32 * QR)      /* inverse-iteration LU + rhs (stride r) */
         + (32 * QR) * (32 * QR) / 8 + 8; /* pivot bytes */
}
__host__ __device__ constexpr size_t eig_small_smem_bytes(int QR) { return (size_t)eig_small_smem_doubles(QR) * 8; }

template <int QR>
__global__ void __launch_bounds__(128 * QR, 1) k_eig_small(const EigTask *__restrict__ tasks, double eps, int *status) {
  constexpr int NW = 4 * QR, UW = 8, MR = 32 * QR;
  extern __shared__ double sh[];
  __shared__ double s_red[32];
  __shared__ double s_bc[8];
  __shared__ int s_int[4];
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  const int m = t.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mp = (m + 8) & ~7;
  double *Hv = sh;
  double *d = Hv + MR * MR, *e = d + (MR + 8), *tau = e + (MR + 8), *e2 = tau + (MR + 8), *lam = e2 + (MR + 8);
  double *zb = lam + (MR + 8);
  double *ws = zb + 2 * MR;                 // inverse-iteration workspace
  double *vbuf = ws, *part = ws + 2 * MR;   // tridiagonalisation scratch (aliases ws)
  if (m <= 0) {
    if (tid == 0) *t.rank_out = 0;
    return;
  }
  if (t.dbg && tid == 0) t.dbg[0] = clock64();
  double a[QR][UW];
#pragma unroll
  for (int q = 0; q < QR; ++q)
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int r = 32 * q + lane, c = UW * warp + u;
      a[q][u] = (r < m && c < m) ? t.G[r + (int64_t)c * m] : 0.0;
    }
  {
    double f = 0.0;
#pragma unroll
    for (int q = 0; q < QR; ++q)
#pragma unroll
      for (int u = 0; u < UW; ++u) f = fma(a[q][u], a[q][u], f);
    f = warp_sum(f);
    if (lane == 0) s_red[warp] = f;
    __syncthreads();
    double fro = 0.0;
    for (int w = 0; w < NW; ++w) fro += s_red[w];
    if (!(fro > 0.0)) {   // G = 0: r = 0 (reading Z4)
      if (tid == 0) *t.rank_out = 0;
      for (int q = tid; q < m; q += blockDim.x) t.sig[q] = 0.0;
      return;
    }
    if (eps == 0.0) {     // eps = 0: nothing truncated, V = I (reading Z3)
      for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x) t.V[q] = ((q % m) == (q / m)) ? 1.0 : 0.0;
      for (int q = tid; q < m; q += blockDim.x) t.sig[q] = 0.0;
      if (tid == 0) *t.rank_out = m;
      return;
    }
  }
  // ---- 1. Householder tridiagonalisation (lower, dsytd2 order) ----
  // v_kk from the (updated) column kk held by its owner warp: v into vbuf[kk & 1]
  // (zero outside rows kk+1..m-1) and Hv[kk m + i], tau[kk], e[kk] = beta.
  auto form_v = [&](int kk) {
    const int u1 = kk % UW;
    double col[QR];
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      double c = a[q][0];
#pragma unroll
      for (int u = 1; u < UW; ++u) c = (u == u1) ? a[q][u] : c;
      col[q] = c;
    }
    double s2 = 0.0;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int r = 32 * q + lane;
      if (r >= kk + 2 && r < m) s2 = fma(col[q], col[q], s2);
    }
    s2 = warp_sum(s2);
    const int rx = kk + 1;
    double xs = col[0];
#pragma unroll
    for (int q = 1; q < QR; ++q) xs = ((rx >> 5) == q) ? col[q] : xs;
    const double x0 = __shfl_sync(0xffffffffu, xs, rx & 31);
    double beta = x0, tk = 0.0, scal = 0.0;
    if (s2 != 0.0) {
      beta = -copysign(sqrt(fma(x0, x0, s2)), x0);
      tk = (beta - x0) * frcp(beta);
      scal = frcp(x0 - beta);
    }
    double *vs = vbuf + (kk & 1) * MR;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int r = 32 * q + lane;
      double v = 0.0;
      if (s2 != 0.0) v = (r == rx) ? 1.0 : ((r > rx && r < m) ? col[q] * scal : 0.0);
      vs[r] = v;
      if (r > kk && r < m) Hv[(int64_t)kk * m + r] = v;
    }
    if (lane == 0) {
      tau[kk] = tk;
      e[kk] = beta;
    }
  };
  if (warp == 0 && m > 2) form_v(0);
  __syncthreads();
  const int ws0 = warp >> 2;   // row group holding this warp's 8 column indices
  long long ph[6] = {0, 0, 0, 0, 0, 0}, pc = clock64();
#define ES_PROF(i)                    \
  if (t.dbg) {                        \
    const long long tn = clock64();   \
    ph[i] += tn - pc;                 \
    pc = tn;                          \
  }
  for (int k = 0; k < m - 2; ++k) {
    const double *vs = vbuf + (k & 1) * MR;
    const double tk = tau[k];
    const int w0 = (k + 1) / UW;   // warps below own only columns <= k (v, w vanish there)
    double vc[UW];
#pragma unroll
    for (int u = 0; u < UW; ++u) vc[u] = vs[UW * warp + u];
    if (warp >= w0) {
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        if (32 * q + 31 <= k) continue;   // rows masked out of p
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int u = 0; u < UW; u += 2) {
          s0 = fma(a[q][u], vc[u], s0);
          s1 = fma(a[q][u + 1], vc[u + 1], s1);
        }
        part[warp * MR + 32 * q + lane] = s0 + s1;
      }
    }
    ES_PROF(0)
    __syncthreads();   // (1) partial products visible
    ES_PROF(1)
    // every warp: p = tau A v for its lanes' rows, p.v, w = p + alpha v
    double vq[QR], wq[QR], pv = 0.0;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int i = 32 * q + lane;
      double s = 0.0;
      if (32 * q + 31 > k)
        for (int w = w0; w < NW; ++w) s += part[w * MR + i];
      const double pi = (i > k && i < m) ? tk * s : 0.0;
      vq[q] = vs[i];
      wq[q] = pi;
      pv = fma(pi, vq[q], pv);
    }
    pv = warp_sum(pv);
    ES_PROF(2)
    const double alpha = -0.5 * tk * pv;
#pragma unroll
    for (int q = 0; q < QR; ++q) wq[q] = fma(alpha, vq[q], wq[q]);
    if (warp >= w0) {
      double wsel = wq[0];
#pragma unroll
      for (int q = 1; q < QR; ++q) wsel = (ws0 == q) ? wq[q] : wsel;
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const double wcu = __shfl_sync(0xffffffffu, wsel, (UW * warp + u) & 31);
#pragma unroll
        for (int q = 0; q < QR; ++q)
          if (32 * q + 31 > k) a[q][u] = fma(-vq[q], wcu, fma(-wq[q], vc[u], a[q][u]));
      }
    }
    ES_PROF(3)
    if (warp == (k + 1) / UW && k + 1 < m - 2) form_v(k + 1);
    ES_PROF(4)
    __syncthreads();   // (2) v_{k+1} visible
    ES_PROF(5)
  }
#undef ES_PROF
  if (t.dbg && lane == 0)
    for (int i = 0; i < 6; ++i) t.dbg[16 + warp * 8 + i] = ph[i];
  // diagonal and last sub-diagonal from the register tiles
#pragma unroll
  for (int q = 0; q < QR; ++q)
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int r = 32 * q + lane, c = UW * warp + u;
      if (r < m && r == c) d[r] = a[q][u];
      if (m >= 2 && r == m - 1 && c == m - 2) e[m - 2] = a[q][u];
    }
  if (tid == 0) {
    e[m - 1] = 0.0;
    if (m >= 2) tau[m - 2] = 0.0;
    tau[m - 1] = 0.0;
  }
  __syncthreads();
  if (t.dbg && tid == 0) t.dbg[1] = clock64();
  // ---- 2. eigenvalues, rank ----
  double bnorm;
  const int r = eig_values_phase(t, eps, m, mp, d, e, e2, lam, s_red, s_bc, s_int, bnorm);
  if (t.dbg && tid == 0) t.dbg[2] = clock64();
  if (r == 0) return;
  // ---- 3. inverse iteration, thread k < r ----
  const double pertol = 10.0 * 2.2e-16 * bnorm;
  if (tid < r) {
    const int k = tid;
    double sft = lam[k];
    for (int q = 1; q <= k && lam[k - q] - lam[k] < pertol; ++q) sft -= pertol;
    const int64_t mr = (int64_t)m * r;
    double *DL = ws + k, *Dv = DL + mr, *DU = Dv + mr, *DU2 = DU + mr, *bb = DU2 + mr;
    unsigned char *pv = reinterpret_cast<unsigned char *>(ws + 5 * mr) + k;
    invit_one(d, e, m, sft, pertol, k, DL, Dv, DU, DU2, bb, pv, r, t.V + (int64_t)k * m);
  }
  __syncthreads();
  if (t.dbg && tid == 0) t.dbg[8] = clock64();
  // ---- 4/5. MGS + back-transformation V = H_0 ... H_{m-3} Z (vectors in registers) ----
  const int per_w = (r + NW - 1) / NW;
  if (per_w > 4) orth_backtr<QR, 8, false>(t.V, Hv, tau, m, r, zb, t.dbg);
  else if (per_w > 2) orth_backtr<QR, 4, false>(t.V, Hv, tau, m, r, zb, t.dbg);
  else if (per_w > 1) orth_backtr<QR, 2, false>(t.V, Hv, tau, m, r, zb, t.dbg);
  else orth_backtr<QR, 1, false>(t.V, Hv, tau, m, r, zb, t.dbg);
  __syncthreads();
  if (t.dbg && tid == 0) t.dbg[3] = t.dbg[4] = clock64();
  (void)status;
}

}  // namespace lorasp
