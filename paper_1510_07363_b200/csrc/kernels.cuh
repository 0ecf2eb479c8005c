// Device kernels of the LoRaSp level sweep (sm_100a, FP64).
//
//  k_leaf_scatter  CSR values -> dense leaf super-node blocks       (P:l.231, l.293)
//  k_copy          block copies / transposes: MergeRedNodes (P:l.298-304)
//                  and the gather of a node's fused pivot record
//  k_gemm          batched tiled DGEMM on task lists: Gram of the
//                  well-separated stack (Eq. lra), R_k = A_k V (P:l.356-359),
//                  Z = L^{-1} C (elimination panel) and the Schur update
//                  -Z_a^T D Z_b scattered into the target blocks (P:l.103-106)
//  k_jacobi        one-sided Jacobi eigen-solver on the Gram matrix, rank by
//                  sigma_k >= eps sigma_0 (Eq. cutOff1, P:l.580-584)
//  k_pivot         signed Cholesky K = L D L^T of the fused (s, b) pivot,
//                  D = diag(I_m, -I_r), and L^{-1}
//  k_apply_fwd/bwd Alg. 3 / Alg. 4 (P:l.445-500) per colour wave
//  Krylov helpers  CSR SpMV, deterministic dots, axpys
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lorasp {

// ---------------------------------------------------------------- copies ----
struct CopyTask {
  const double *src;
  double *dst;
  int lds, ldd, rows, cols;
  int mode;           // 0: copy, 1: fill the rows x cols rectangle with alpha,
                      // 2: alpha on the diagonal and 0 elsewhere (rows x cols)
  int trans;          // mode 0: dst(i,j) = alpha * src(j,i)
  double alpha;
};

__global__ void __launch_bounds__(256) k_copy(const CopyTask *__restrict__ tasks) {
  const CopyTask t = tasks[blockIdx.x];
  if (t.rows <= 0 || t.cols <= 0) return;
  const int64_t tot = (int64_t)t.rows * t.cols;
  if (t.mode != 0) {
    for (int64_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      int i = (int)(idx % t.rows), j = (int)(idx / t.rows);
      t.dst[i + (int64_t)j * t.ldd] = (t.mode == 1 || i == j) ? t.alpha : 0.0;
    }
    return;
  }
  if (!t.trans) {
    for (int64_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      int i = (int)(idx % t.rows), j = (int)(idx / t.rows);
      t.dst[i + (int64_t)j * t.ldd] = t.alpha * t.src[i + (int64_t)j * t.lds];
    }
  } else {
    // transpose through shared memory 32x32 tiles (coalesced on both sides)
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // blockDim = 256 -> ty 0..7
    for (int bj = 0; bj < t.cols; bj += 32)
      for (int bi = 0; bi < t.rows; bi += 32) {
        for (int q = ty; q < 32; q += 8) {
          int j = bj + tx, i = bi + q;   // src(j, i): j contiguous in src
          tile[q][tx] = (j < t.cols && i < t.rows) ? t.src[j + (int64_t)i * t.lds] : 0.0;
        }
        __syncthreads();
        for (int q = ty; q < 32; q += 8) {
          int i = bi + tx, j = bj + q;
          if (i < t.rows && j < t.cols) t.dst[i + (int64_t)j * t.ldd] = t.alpha * tile[tx][q];
        }
        __syncthreads();
      }
  }
}

__global__ void k_leaf_scatter(const double *__restrict__ vals, const int64_t *__restrict__ dest,
                               int64_t nnz, double *__restrict__ base) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = dest[k];
    if (d >= 0) base[d] = vals[k];
  }
}

// ------------------------------------------------------------------ GEMM ----
// C(tile) = beta*C + sum_seg alpha_seg * op(A_seg) op(B_seg) on a 64x64 tile.
struct GemmSeg {
  const double *A, *B;
  int lda, ldb, K;
  double alpha;
};
struct GemmTask {
  double *C;
  int ldc, M, N;     // full logical extents of C
  int tm, tn;        // tile origin
  int ta, tb, tc;    // op(A) = A^T, op(B) = B^T, C stored transposed
  int beta;          // 0: overwrite, 1: accumulate
  int seg0, nseg;
};

constexpr int GT = 64, GK = 16;

__global__ void __launch_bounds__(256) k_gemm(const GemmTask *__restrict__ tasks,
                                              const GemmSeg *__restrict__ segs) {
  const GemmTask t = tasks[blockIdx.x];
  __shared__ double As[GK][GT + 1];
  __shared__ double Bs[GK][GT + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  for (int s = 0; s < t.nseg; ++s) {
    const GemmSeg g = segs[t.seg0 + s];
    double accs[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) accs[a][b] = 0.0;
    for (int k0 = 0; k0 < g.K; k0 += GK) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int idx = tid + 256 * q;
        int i, kk;
        if (!t.ta) { i = idx & 63; kk = idx >> 6; } else { kk = idx & 15; i = idx >> 4; }
        int gi = t.tm + i, gk = k0 + kk;
        double v = 0.0;
        if (gi < t.M && gk < g.K)
          v = t.ta ? g.A[gk + (int64_t)gi * g.lda] : g.A[gi + (int64_t)gk * g.lda];
        As[kk][i] = v;
        int j;
        if (!t.tb) { kk = idx & 15; j = idx >> 4; } else { j = idx & 63; kk = idx >> 6; }
        int gj = t.tn + j;
        gk = k0 + kk;
        v = 0.0;
        if (gj < t.N && gk < g.K)
          v = t.tb ? g.B[gj + (int64_t)gk * g.ldb] : g.B[gk + (int64_t)gj * g.ldb];
        Bs[kk][j] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < GK; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][tx + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][ty + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) accs[a][b] = fma(av[a], bv[b], accs[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(g.alpha, accs[a][b], acc[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int i = t.tm + tx + 16 * a, j = t.tn + ty + 16 * b;
      if (i < t.M && j < t.N) {
        double *p = t.tc ? &t.C[j + (int64_t)i * t.ldc] : &t.C[i + (int64_t)j * t.ldc];
        *p = t.beta ? (*p + acc[a][b]) : acc[a][b];
      }
    }
}

// ---------------------------------------------------------------- Jacobi ----
// One-sided (Hestenes) Jacobi on the symmetric PSD Gram matrix G = M^T M:
// right rotations Y <- Y J until the columns of Y are mutually orthogonal;
// then Y = G V = V diag(lambda): ||y_k|| = lambda_k = sigma_k^2 and
// y_k / ||y_k|| = v_k, without accumulating V.  Cyclic round-robin pairs, one
// warp per pair.  Rank r = #{sigma_k >= eps sigma_0}; eps = 0 keeps every
// direction (reading Z3): V = I_m, r = m (r = 0 if G = 0, reading Z4).
struct EigTask {
  const double *G;   // m x m, ld m
  double *V;         // out: m x r (ld m), columns sorted by sigma descending
  double *sig;       // out: m sigma values, descending
  double *work;      // global scratch m x m when it does not fit shared memory
  int m;
  int node;          // cluster id (for status)
  int *rank_out;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int EIG_MAX_SWEEPS = 60;

__global__ void __launch_bounds__(512) k_jacobi(const EigTask *__restrict__ tasks, double eps,
                                                int smem_cap_doubles, int *status) {
  extern __shared__ double sh[];
  const EigTask t = tasks[blockIdx.x];
  const int m = t.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // shared layout: [lam (m) | rankpos (m ints as doubles) | X (m*m if it fits)]
  double *lam = sh;
  int *rk = reinterpret_cast<int *>(sh + m);
  double *X = ((int64_t)m * m + 2 * m <= smem_cap_doubles) ? sh + 2 * m : t.work;
  __shared__ int s_flag;
  __shared__ double s_red[32];
  for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x) X[q] = t.G[q];
  __syncthreads();
  // Frobenius norm (zero test)
  double fro = 0;
  for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x) fro += X[q] * X[q];
  fro = warp_sum(fro);
  if (lane == 0) s_red[warp] = fro;
  __syncthreads();
  if (tid == 0) {
    double s = 0;
    for (int w = 0; w < nw; ++w) s += s_red[w];
    s_flag = (s > 0.0);
  }
  __syncthreads();
  if (!s_flag) {
    if (tid == 0) *t.rank_out = 0;
    for (int q = tid; q < m; q += blockDim.x) t.sig[q] = 0.0;
    return;
  }
  if (eps == 0.0) {  // nothing truncated: any orthonormal basis is exact
    for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x)
      t.V[q] = ((q % m) == (q / m)) ? 1.0 : 0.0;
    for (int q = tid; q < m; q += blockDim.x) t.sig[q] = 0.0;
    if (tid == 0) *t.rank_out = m;
    return;
  }
  const int n2 = m + (m & 1);
  const double tol = fmax(1e-14, 2.3e-16 * m);
  int sweep = 0;
  for (; sweep < EIG_MAX_SWEEPS; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < n2 - 1; ++step) {
      for (int j = warp; j < n2 / 2; j += nw) {
        int pp = (j == 0) ? 0 : 1 + (j - 1 + step) % (n2 - 1);
        int qp = n2 - 1 - j;
        int qq = 1 + (qp - 1 + step) % (n2 - 1);
        int p = pp, q = qq;
        if (p >= m || q >= m) continue;
        double *xp = X + (int64_t)p * m, *xq = X + (int64_t)q * m;
        double al = 0, be = 0, ga = 0;
        for (int r = lane; r < m; r += 32) {
          double a = xp[r], b = xq[r];
          al = fma(a, a, al);
          be = fma(b, b, be);
          ga = fma(a, b, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al == 0.0 || be == 0.0) continue;
        if (fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
        double zeta = (be - al) / (2.0 * ga);
        double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int r = lane; r < m; r += 32) {
          double a = xp[r], b = xq[r];
          xp[r] = c * a - s * b;
          xq[r] = s * a + c * b;
        }
        rotated = 1;
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  if (sweep == EIG_MAX_SWEEPS && tid == 0) {
    atomicCAS(&status[0], 0, -4);
    status[1] = t.node;
  }
  // lambda_k = ||y_k||
  for (int k = warp; k < m; k += nw) {
    double s = 0;
    const double *xk = X + (int64_t)k * m;
    for (int r = lane; r < m; r += 32) s = fma(xk[r], xk[r], s);
    s = warp_sum(s);
    if (lane == 0) lam[k] = sqrt(s);
  }
  __syncthreads();
  // sort descending (stable by index): position of k
  for (int k = tid; k < m; k += blockDim.x) {
    double lk = lam[k];
    int pos = 0;
    for (int j = 0; j < m; ++j) {
      double lj = lam[j];
      pos += (lj > lk) || (lj == lk && j < k);
    }
    rk[k] = pos;
  }
  __syncthreads();
  double lam0 = 0;
  for (int k = 0; k < m; ++k) lam0 = fmax(lam0, lam[k]);
  const double sig0 = sqrt(lam0);
  int r = 0;
  for (int k = 0; k < m; ++k) r += (sqrt(lam[k]) >= eps * sig0);
  for (int k = tid; k < m; k += blockDim.x) t.sig[rk[k]] = sqrt(lam[k]);
  for (int k = warp; k < m; k += nw) {
    int pk = rk[k];
    if (pk >= r) continue;
    double inv = 1.0 / lam[k];
    const double *xk = X + (int64_t)k * m;
    double *vk = t.V + (int64_t)pk * m;
    for (int q = lane; q < m; q += 32) vk[q] = xk[q] * inv;
  }
  if (tid == 0) *t.rank_out = r;
}

// ----------------------------------------------------------------- pivot ----
// Fused pivot of (s, b): K = [[S, V], [V^T, 0]] (n = m + r) factored as
// K = L D L^T with D = diag(I_m, -I_r) (Cholesky of S, then of
// W = V^T S^{-1} V for the black node, P:l.396-399), then overwritten by
// L^{-1} (lower, strict upper zeroed).  Works in shared memory when n^2 fits.
struct PivTask {
  double *F;  // n x n at ld
  int ld, m, r, node;
};

__global__ void __launch_bounds__(512) k_pivot(const PivTask *__restrict__ tasks,
                                               int smem_cap_doubles, int *status) {
  extern __shared__ double sh[];
  const PivTask t = tasks[blockIdx.x];
  const int n = t.m + t.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ int s_fail;
  const bool in_smem = (int64_t)n * n + n <= smem_cap_doubles;
  double *tmp = sh;  // n
  double *A;
  int lda;
  if (in_smem) {
    A = sh + n;
    lda = n;
    for (int64_t q = tid; q < (int64_t)n * n; q += blockDim.x) {
      int i = (int)(q % n), j = (int)(q / n);
      A[q] = (i >= j) ? t.F[i + (int64_t)j * t.ld] : 0.0;
    }
  } else {
    A = t.F;
    lda = t.ld;
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  // signed right-looking Cholesky
  for (int k = 0; k < n; ++k) {
    const double d = (k < t.m) ? 1.0 : -1.0;
    const double v = A[k + (int64_t)k * lda] * d;
    if (!(v > 0.0) || !isfinite(v)) {  // uniform across threads
      if (tid == 0) {
        s_fail = 1;
        if (atomicCAS(&status[0], 0, -3) == 0) status[1] = t.node;
      }
      break;
    }
    const double lkk = sqrt(v);
    const double sc = 1.0 / (d * lkk);
    __syncthreads();
    for (int i = k + 1 + tid; i < n; i += blockDim.x) A[i + (int64_t)k * lda] *= sc;
    __syncthreads();
    if (tid == 0) A[k + (int64_t)k * lda] = lkk;
    for (int j = k + 1 + warp; j < n; j += nw) {
      const double ljk = A[j + (int64_t)k * lda] * d;
      double *cj = A + (int64_t)j * lda;
      const double *ck = A + (int64_t)k * lda;
      for (int i = j + lane; i < n; i += 32) cj[i] = fma(-ck[i], ljk, cj[i]);
    }
    __syncthreads();
  }
  if (s_fail) return;
  // in-place inverse of the lower-triangular L (column j from n-1 down to 0)
  for (int j = n - 1; j >= 0; --j) {
    for (int i = j + 1 + tid; i < n; i += blockDim.x) tmp[i] = A[i + (int64_t)j * lda];
    __syncthreads();
    const double ajj = 1.0 / A[j + (int64_t)j * lda];
    for (int i = j + 1 + tid; i < n; i += blockDim.x) {
      double s = 0;
      for (int k = j + 1; k <= i; ++k) s = fma(A[i + (int64_t)k * lda], tmp[k], s);
      A[i + (int64_t)j * lda] = -ajj * s;
    }
    __syncthreads();
    if (tid == 0) A[j + (int64_t)j * lda] = ajj;
    __syncthreads();
  }
  // write back L^{-1} with the strict upper triangle zeroed
  for (int64_t q = tid; q < (int64_t)n * n; q += blockDim.x) {
    int i = (int)(q % n), j = (int)(q / n);
    double v = (i >= j) ? A[i + (int64_t)j * lda] : 0.0;
    t.F[i + (int64_t)j * t.ld] = v;
  }
}

// ----------------------------------------------------------------- apply ----
// Forward (Alg. 3) and backward (Alg. 4) over the fused records
//   F = [ L^{-1} (n x n) | Z (n x W) ],  Z = L^{-1} C,  C = coupling to T.
// forward:  y = L^{-1} [rhs_s; 0];  rhs_q -= Z_q^T D y           (q in T)
// backward: u = y - Z x_T;  [x_s; x_b] = L^{-T} D u               (P:l.487-495)
struct ApNode {
  const double *F;
  double *y;       // n doubles, kept between the two passes
  int64_t off_s;   // vector offset of Var/RHS(s)
  int m, r, W;
  int seg0, nseg;
};
struct ApSeg {
  int64_t voff;   // vector offset of the target's Var/RHS
  int w, zc;      // width, column offset inside Z
};

__global__ void __launch_bounds__(256) k_apply_fwd(const ApNode *__restrict__ nodes,
                                                   const ApSeg *__restrict__ segs,
                                                   double *__restrict__ vec) {
  extern __shared__ double sh[];
  const ApNode nd = nodes[blockIdx.x];
  const int n = nd.m + nd.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *rhs = sh;      // m
  double *dy = sh + nd.m;  // n
  for (int i = tid; i < nd.m; i += blockDim.x) rhs[i] = vec[nd.off_s + i];
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    double s = 0;
    const int kmax = min(i, nd.m - 1);
    for (int k = 0; k <= kmax; ++k) s = fma(nd.F[i + (int64_t)k * n], rhs[k], s);
    nd.y[i] = s;
    dy[i] = (i < nd.m) ? s : -s;
  }
  __syncthreads();
  const double *Z = nd.F + (int64_t)n * n;
  for (int sg = 0; sg < nd.nseg; ++sg) {
    const ApSeg S = segs[nd.seg0 + sg];
    for (int j = warp; j < S.w; j += nw) {
      const double *zc = Z + (int64_t)(S.zc + j) * n;
      double s = 0;
      for (int k = lane; k < n; k += 32) s = fma(zc[k], dy[k], s);
      s = warp_sum(s);
      if (lane == 0) vec[S.voff + j] -= s;
    }
  }
}

__global__ void __launch_bounds__(256) k_apply_bwd(const ApNode *__restrict__ nodes,
                                                   const ApSeg *__restrict__ segs,
                                                   double *__restrict__ vec) {
  extern __shared__ double sh[];
  const ApNode nd = nodes[blockIdx.x];
  const int n = nd.m + nd.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *u = sh;           // n
  double *xt = sh + n;      // W
  for (int sg = 0; sg < nd.nseg; ++sg) {
    const ApSeg S = segs[nd.seg0 + sg];
    for (int j = tid; j < S.w; j += blockDim.x) xt[S.zc + j] = vec[S.voff + j];
  }
  __syncthreads();
  const double *Z = nd.F + (int64_t)n * n;
  for (int k = tid; k < n; k += blockDim.x) {
    double s = nd.y[k];
    for (int j = 0; j < nd.W; ++j) s = fma(-Z[k + (int64_t)j * n], xt[j], s);
    u[k] = (k < nd.m) ? s : -s;  // D u
  }
  __syncthreads();
  for (int i = warp; i < nd.m; i += nw) {
    const double *li = nd.F + (int64_t)i * n;  // column i of L^{-1}: rows >= i
    double s = 0;
    for (int k = i + lane; k < n; k += 32) s = fma(li[k], u[k], s);
    s = warp_sum(s);
    if (lane == 0) vec[nd.off_s + i] = s;
  }
}

__global__ void k_set_rhs(const double *__restrict__ b, const int64_t *__restrict__ perm, int64_t n,
                          double *__restrict__ vec) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    vec[perm[q]] = b[q];
}
__global__ void k_get_x(const double *__restrict__ vec, const int64_t *__restrict__ perm, int64_t n,
                        double *__restrict__ x) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    x[q] = vec[perm[q]];
}

// ---------------------------------------------------------------- Krylov ----
__global__ void k_spmv(int64_t n, const int64_t *__restrict__ rp, const int64_t *__restrict__ ci,
                       const double *__restrict__ va, const double *__restrict__ x,
                       double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s = fma(va[k], x[ci[k]], s);
    y[i] = s;
  }
}

// deterministic two-pass dot: fixed grid, per-block partials, final single block
constexpr int DOT_BLOCKS = 296;
__global__ void __launch_bounds__(256) k_dot_partial(int64_t n, const double *__restrict__ a,
                                                     const double *__restrict__ b,
                                                     double *__restrict__ part) {
  __shared__ double red[8];
  double s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void k_dot_final(const double *__restrict__ part, int np, double *__restrict__ out) {
  __shared__ double red[8];
  double s = 0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    *out = t;
  }
}
// y = a*x + b*y
__global__ void k_axpby(int64_t n, double a, const double *__restrict__ x, double b,
                        double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}
// z = x - y
__global__ void k_sub(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                      double *__restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = x[i] - y[i];
}

}  // namespace lorasp
