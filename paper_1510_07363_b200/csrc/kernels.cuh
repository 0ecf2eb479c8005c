// Device kernels of the LoRaSp level sweep (sm_100a, FP64).
//
//  k_leaf_scatter     CSR values -> dense leaf super-node blocks    (P:l.231, l.293)
//  k_copy             block copies / transposes: MergeRedNodes (P:l.298-304)
//                     and the gather of a node's fused pivot record
//  k_gemm2_dmma       batched tiled DGEMM on task lists, FP64 tensor cores (DMMA;
//                     k_gemm2 = the DFMA variant, kept for the per-shape
//                     comparison hook lorasp_test_gemm): Gram of the
//                     well-separated stack (Eq. lra), R_k = A_k V (P:l.356-359),
//                     Z = L^{-1} C (elimination panel), the Schur update
//                     -Z_a^T D Z_b scattered into the target blocks (P:l.103-106)
//  Compress eigen-solver (sigma_k = sqrt(lambda_k(G)), rank sigma_k >= eps sigma_0,
//  Eq. cutOff1, P:l.580-584):
//    k_tridiag_reg    Householder tridiagonalisation, m <= 128, G in registers
//    k_tridiag_cl     the same over a thread-block cluster, 128 < m <= 512
//    k_eig_t          eigenvalues (Sturm multisection), inverse iteration, MGS,
//                     back-transformation (generic m or after the kernels above)
//    k_invit_multi / k_orth_bgs / k_backtr_multi   the same steps split over CTAs
//                     for 128 < m <= 512 (ranks ~0.6 m there)
//  Fused (s, b) pivot (P:l.396-399, P:l.101-106):
//    k_pivot_blk      signed Cholesky K = L diag(I_m, -I_r) L^T + L^{-1}, n <= 160
//    k_pivot_lu_blk / k_pivot_lu   LU path (LU, L^{-1} P and U^{-T}; partial
//                     pivoting in k_pivot_lu once the no-pivot multipliers grow)
//  k_apply_fwd/bwd    Alg. 3 / Alg. 4 (P:l.445-500) per colour wave (+ the split
//                     k_apply_fwd_y/_z, k_apply_bwd_z/_l for few large records)
//  Krylov helpers     CSR SpMV, deterministic dots, axpys
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace lorasp {

// Programmatic dependent launch (the factor sweep's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): every such kernel lets
// its successor be scheduled at once and waits for its predecessor's memory
// before touching anything.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_trigger();
  pdl_wait();
}

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
  pdl_trigger();
  const CopyTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  if (t.rows <= 0 || t.cols <= 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (t.mode != 0) {
    for (int j = warp; j < t.cols; j += nw)
      for (int i = lane; i < t.rows; i += 32)
        t.dst[i + (int64_t)j * t.ldd] = (t.mode == 1 || i == j) ? t.alpha : 0.0;
    return;
  }
  if (!t.trans) {
    for (int j = warp; j < t.cols; j += nw)
      for (int i = lane; i < t.rows; i += 32)
        t.dst[i + (int64_t)j * t.ldd] = t.alpha * t.src[i + (int64_t)j * t.lds];
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
  pdl_enter();
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
  int tnw;           // k_gemm2 tile width: 32 for narrow products (N <= 32), else 64 (0 = 64)
};

constexpr int GT = 64, GK = 32;

// k_gemm2: tile GEMM tasks (C tile 64 x 64 = sum_seg alpha op(A)
// op(B), beta accumulate, tc = store transposed), 128 threads with 4 x 8
// accumulators each (32 FMAs per 12 shared loads), cp.async double-buffered
// 16-deep K chunks (no staging registers), alpha folded into the A fragment
// (one accumulator set across segments).  Up to 4 CTAs per SM.
constexpr int G2K = 16;
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, const void *gbase, bool pred) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;   // 0: zero-fill (the source, a valid global address, is not read)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(pred ? gmem : gbase), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One 64 x (8 NB) tile of a k_gemm2 task (NB = 8: 64 columns, NB = 4: 32).
template <int NB>
__device__ __forceinline__ void gemm2_tile(const GemmTask &t, const GemmSeg *__restrict__ segs,
                                           double (*As)[G2K][GT + 1], double (*Bs)[G2K][GT + 1]) {
  constexpr int TN = 8 * NB;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;   // rows tx + 16 a, columns ty + 8 b
  double acc[4][NB];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[a][b] = 0.0;

  for (int s = 0; s < t.nseg; ++s) {
    const GemmSeg g = segs[t.seg0 + s];
    if (g.K <= 0) continue;
    auto load = [&](int k0, int st) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int idx = tid + 128 * q;   // A: 64 x 16
        int i, kk;
        if (!t.ta) { i = idx & 63; kk = idx >> 6; } else { kk = idx & 15; i = idx >> 4; }
        const int gi = t.tm + i, gk = k0 + kk;
        cp_async8(&As[st][kk][i], t.ta ? g.A + (gk + (int64_t)gi * g.lda) : g.A + (gi + (int64_t)gk * g.lda), g.A,
                  gi < t.M && gk < g.K);
      }
#pragma unroll
      for (int q = 0; q < TN / 8; ++q) {
        const int idx = tid + 128 * q;   // B: 16 x TN
        int j, kk;
        if (!t.tb) { kk = idx & 15; j = idx >> 4; } else { j = idx % TN; kk = idx / TN; }
        const int gj = t.tn + j, gk = k0 + kk;
        cp_async8(&Bs[st][kk][j], t.tb ? g.B + (gj + (int64_t)gk * g.ldb) : g.B + (gk + (int64_t)gj * g.ldb), g.B,
                  gj < t.N && gk < g.K);
      }
      cp_async_commit();
    };
    const double alpha = g.alpha;
    const int nch = (g.K + G2K - 1) / G2K;
    load(0, 0);
    for (int c = 0; c < nch; ++c) {
      if (c + 1 < nch) {
        load((c + 1) * G2K, (c + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const int st = c & 1;
      // alpha = +-1 (every segment the sweep issues) rides on the FMA's operand
      // negation for free; other values scale the A fragment
      auto chunk = [&](auto sgn) {
#pragma unroll
        for (int kk = 0; kk < G2K; ++kk) {
          double av[4], bv[NB];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const double x = As[st][kk][tx + 16 * a];
            av[a] = decltype(sgn)::value == 0 ? alpha * x : (decltype(sgn)::value > 0 ? x : -x);
          }
#pragma unroll
          for (int b = 0; b < NB; ++b) bv[b] = Bs[st][kk][ty + 8 * b];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
      };
      if (alpha == 1.0) chunk(std::integral_constant<int, 1>{});
      else if (alpha == -1.0) chunk(std::integral_constant<int, -1>{});
      else chunk(std::integral_constant<int, 0>{});
      __syncthreads();   // stage st is refilled by the load two chunks ahead
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = t.tm + tx + 16 * a, j = t.tn + ty + 8 * b;
      if (i < t.M && j < t.N) {
        double *p = t.tc ? &t.C[j + (int64_t)i * t.ldc] : &t.C[i + (int64_t)j * t.ldc];
        *p = t.beta ? (*p + acc[a][b]) : acc[a][b];
      }
    }
}

__global__ void __launch_bounds__(128, 4) k_gemm2(const GemmTask *__restrict__ tasks,
                                                const GemmSeg *__restrict__ segs) {
  __shared__ __align__(16) double As[2][G2K][GT + 1];
  __shared__ __align__(16) double Bs[2][G2K][GT + 1];
  pdl_trigger();
  const GemmTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  if (t.tnw == 32) gemm2_tile<4>(t, segs, As, Bs);
  else gemm2_tile<8>(t, segs, As, Bs);
}

// k_gemm2_dmma: the same tasks on the FP64 tensor cores (DMMA, mma.sync
// m8n8k4 .f64; north_star item 3).  Identical staging (cp.async double-buffered
// 16-deep K chunks in shared memory); the 4 warps split the 64 x TN tile 2 x 2,
// each warp owning 4 x (TN/16) 8 x 8 accumulator fragments.  Per 4-deep k step a
// lane loads 4 A and TN/16 B fragment doubles for 4 x TN/16 DMMAs (256 / 128
// flops per loaded double vs 5.3 for the DFMA tile).  Fragment layout (PTX
// m8n8k4 .f64): A[g][t], B[t][g], C[g][2t + {0, 1}] with g = lane >> 2,
// t = lane & 3.  Rounding differs from k_gemm2 (hardware accumulation order).
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// Shared tiles of the DMMA kernel.  An operand whose rows are contiguous in
// memory (A not transposed, B transposed) is staged k-major [16][GLD] (row
// stride 72 doubles); one whose K is contiguous (A transposed, B not -- the
// Gram, Schur and most products) is staged row-major [64][GLK] (row stride 20
// doubles).  Both strides keep 16-byte aligned pairs for the 16-byte async
// copies and put the fragment reads of lanes (g, tq) on 2 wavefronts, the
// minimum for 32 doubles.
constexpr int GLD = 72, GLK = 20, GSTAGE = 64 * GLK;   // 1280 >= 16 x 72
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, const void *gbase, int bytes) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(bytes ? gmem : gbase), "r"(bytes)
               : "memory");
}
// AK: op(A) tile stored [i][k] (t.ta); BK: op(B) tile stored [j][k] (!t.tb)
template <int NB, bool AK, bool BK>
__device__ __forceinline__ void gemm2_tile_dmma(const GemmTask &t, const GemmSeg *__restrict__ segs,
                                                double (*As)[GSTAGE], double (*Bs)[GSTAGE]) {
  constexpr int TN = 8 * NB, CB = TN / 16;   // column fragments per warp
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 1, wc = warp >> 1;   // warp sub-tile: rows 32 wr.., cols (TN/2) wc..
  const int g = lane >> 2, tq = lane & 3;
  double acc[4][CB][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int s = 0; s < t.nseg; ++s) {
    const GemmSeg gs = segs[t.seg0 + s];
    if (gs.K <= 0) continue;
    // 16-byte copies when the contiguous pairs are 16-byte aligned
    const bool a16 = (gs.lda & 1) == 0 && ((uintptr_t)gs.A & 15) == 0;
    const bool b16 = (gs.ldb & 1) == 0 && ((uintptr_t)gs.B & 15) == 0;
    auto load = [&](int k0, int st) {
      if constexpr (AK) {   // A(gk, gi) at A + gk + gi lda
        if (a16) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = tid + 128 * q, i = idx >> 3, kk = 2 * (idx & 7);
            const int gi = t.tm + i, gk = k0 + kk;
            const int nb = (gi < t.M) ? (gk + 1 < gs.K ? 16 : (gk < gs.K ? 8 : 0)) : 0;
            cp_async16(&As[st][i * GLK + kk], gs.A + (gk + (int64_t)gi * gs.lda), gs.A, nb);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int idx = tid + 128 * q, kk = idx & 15, i = idx >> 4;
            const int gi = t.tm + i, gk = k0 + kk;
            cp_async8(&As[st][i * GLK + kk], gs.A + (gk + (int64_t)gi * gs.lda), gs.A, gi < t.M && gk < gs.K);
          }
        }
      } else {   // A(gi, gk) at A + gi + gk lda
        if (a16) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = tid + 128 * q, i = 2 * (idx & 31), kk = idx >> 5;
            const int gi = t.tm + i, gk = k0 + kk;
            const int nb = (gk < gs.K) ? (gi + 1 < t.M ? 16 : (gi < t.M ? 8 : 0)) : 0;
            cp_async16(&As[st][kk * GLD + i], gs.A + (gi + (int64_t)gk * gs.lda), gs.A, nb);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int idx = tid + 128 * q, i = idx & 63, kk = idx >> 6;
            const int gi = t.tm + i, gk = k0 + kk;
            cp_async8(&As[st][kk * GLD + i], gs.A + (gi + (int64_t)gk * gs.lda), gs.A, gi < t.M && gk < gs.K);
          }
        }
      }
      if constexpr (BK) {   // B(gk, gj) at B + gk + gj ldb
        if (b16) {
#pragma unroll
          for (int q = 0; q < TN / 16; ++q) {
            const int idx = tid + 128 * q, j = idx >> 3, kk = 2 * (idx & 7);
            const int gj = t.tn + j, gk = k0 + kk;
            const int nb = (gj < t.N) ? (gk + 1 < gs.K ? 16 : (gk < gs.K ? 8 : 0)) : 0;
            cp_async16(&Bs[st][j * GLK + kk], gs.B + (gk + (int64_t)gj * gs.ldb), gs.B, nb);
          }
        } else {
#pragma unroll
          for (int q = 0; q < TN / 8; ++q) {
            const int idx = tid + 128 * q, kk = idx & 15, j = idx >> 4;
            const int gj = t.tn + j, gk = k0 + kk;
            cp_async8(&Bs[st][j * GLK + kk], gs.B + (gk + (int64_t)gj * gs.ldb), gs.B, gj < t.N && gk < gs.K);
          }
        }
      } else {   // B(gj, gk) at B + gj + gk ldb
        if (b16) {
#pragma unroll
          for (int q = 0; q < TN / 16; ++q) {
            const int idx = tid + 128 * q, j = 2 * (idx % (TN / 2)), kk = idx / (TN / 2);
            const int gj = t.tn + j, gk = k0 + kk;
            const int nb = (gk < gs.K) ? (gj + 1 < t.N ? 16 : (gj < t.N ? 8 : 0)) : 0;
            cp_async16(&Bs[st][kk * GLD + j], gs.B + (gj + (int64_t)gk * gs.ldb), gs.B, nb);
          }
        } else {
#pragma unroll
          for (int q = 0; q < TN / 8; ++q) {
            const int idx = tid + 128 * q, j = idx % TN, kk = idx / TN;
            const int gj = t.tn + j, gk = k0 + kk;
            cp_async8(&Bs[st][kk * GLD + j], gs.B + (gj + (int64_t)gk * gs.ldb), gs.B, gj < t.N && gk < gs.K);
          }
        }
      }
      cp_async_commit();
    };
    // alpha = +-1 (every product of the sweep): the sign goes on the
    // accumulators around the segment (exact), no multiply per fragment
    const double alpha = gs.alpha;
    const bool neg = alpha == -1.0, unit = neg || alpha == 1.0;
    if (neg)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < CB; ++b) {
          acc[a][b][0] = -acc[a][b][0];
          acc[a][b][1] = -acc[a][b][1];
        }
    const int nch = (gs.K + G2K - 1) / G2K;
    load(0, 0);
    for (int c = 0; c < nch; ++c) {
      if (c + 1 < nch) {
        load((c + 1) * G2K, (c + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double *Ast = As[c & 1], *Bst = Bs[c & 1];
#pragma unroll
      for (int k4 = 0; k4 < G2K; k4 += 4) {
        double af[4], bf[CB];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = 32 * wr + 8 * a + g, k = k4 + tq;
          const double v = AK ? Ast[i * GLK + k] : Ast[k * GLD + i];
          af[a] = unit ? v : alpha * v;
        }
#pragma unroll
        for (int b = 0; b < CB; ++b) {
          const int j = (TN / 2) * wc + 8 * b + g, k = k4 + tq;
          bf[b] = BK ? Bst[j * GLK + k] : Bst[k * GLD + j];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < CB; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
      __syncthreads();
    }
    if (neg)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < CB; ++b) {
          acc[a][b][0] = -acc[a][b][0];
          acc[a][b][1] = -acc[a][b][1];
        }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = t.tm + 32 * wr + 8 * a + g, j = t.tn + (TN / 2) * wc + 8 * b + 2 * tq + e;
        if (i < t.M && j < t.N) {
          double *p = t.tc ? &t.C[j + (int64_t)i * t.ldc] : &t.C[i + (int64_t)j * t.ldc];
          *p = t.beta ? (*p + acc[a][b][e]) : acc[a][b][e];
        }
      }
}

__global__ void __launch_bounds__(128, 4) k_gemm2_dmma(const GemmTask *__restrict__ tasks,
                                                     const GemmSeg *__restrict__ segs) {
  __shared__ __align__(16) double As[2][GSTAGE];
  __shared__ __align__(16) double Bs[2][GSTAGE];
  pdl_trigger();
  const GemmTask t = tasks[blockIdx.x];
  pdl_wait();
  const int sel = (t.tnw == 32 ? 4 : 0) + (t.ta ? 2 : 0) + (t.tb ? 0 : 1);
  switch (sel) {
    case 0: gemm2_tile_dmma<8, false, false>(t, segs, As, Bs); break;
    case 1: gemm2_tile_dmma<8, false, true>(t, segs, As, Bs); break;
    case 2: gemm2_tile_dmma<8, true, false>(t, segs, As, Bs); break;
    case 3: gemm2_tile_dmma<8, true, true>(t, segs, As, Bs); break;
    case 4: gemm2_tile_dmma<4, false, false>(t, segs, As, Bs); break;
    case 5: gemm2_tile_dmma<4, false, true>(t, segs, As, Bs); break;
    case 6: gemm2_tile_dmma<4, true, false>(t, segs, As, Bs); break;
    default: gemm2_tile_dmma<4, true, true>(t, segs, As, Bs); break;
  }
}

struct EigTask {
  const double *G;   // m x m, ld m
  double *V;         // out: m x r (ld m), columns sorted by sigma descending
  double *sig;       // out: m sigma values, descending
  double *work;      // global scratch m x m when it does not fit shared memory
  int m;
  int node;          // cluster id (for status)
  int *rank_out;
  long long *dbg;    // optional phase timestamps (test hook), may be null
  // Frobenius rule (f2, Eq. curOff6 P:l.756-761, reading F2): device scalar
  // D^2 = ||all levels below||_F^2; nullptr = the relative-sigma rule Eq. cutOff1.
  // frob_w: energy of the oracle's stack [A; B] per unit of this stack's (SPD path
  // stacks only A: 2; LU path: 1)
  const double *frob;
  double frob_w;
};

// FP64 division is a long software sequence on sm_100a (~430 cycles of latency
// measured, tools/micro/fp64lat.cu); the reciprocal from MUFU.RCP64H plus two
// Newton steps costs ~50 cycles and matched IEEE 1/x on every tested input.
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 1 / sqrt(x) for x > 0: MUFU.RSQ64H approximation + two Newton steps
// (y <- y (3 - x y^2) / 2); replaces the IEEE sqrt + reciprocal pair on the
// pivot kernels' dependent chain (one per column)
__device__ __forceinline__ double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}



// ------------------------------------------------- tridiagonal eigen-solver ----
// Symmetric eigen-decomposition of the Gram matrix G = M^T M for Compress
// (sigma_k = sqrt(lambda_k), P:l.333-359) in O(m^3) with few sequential steps:
//   1. Householder tridiagonalisation Q^T G Q = T (lower, LAPACK sytd2 form);
//   2. eigenvalues of T by Sturm-count multisection (one warp per eigenvalue,
//      32 points per round): lambda_0 first, then only the candidates with
//      lambda >= (eps sigma_0)^2 / 4 (a superset of the kept ones);
//   3. rank r = #{sqrt(lambda_k) >= eps sqrt(lambda_0)} (Eq. cutOff1);
//   4. eigenvectors of T for the r kept eigenvalues by inverse iteration
//      (pivoted tridiagonal LU, 3 sweeps, re-orthogonalised inside clusters);
//   5. back-transformation V = Q Z.
// eps = 0 keeps every direction (reading Z3): V = I_m, r = m.
struct EigScratch {
  double *work;  // >= 7 m^2 doubles of global scratch per task
};

__device__ __forceinline__ int sturm_count(const double *__restrict__ d, const double *__restrict__ e2,
                                           int m, double x, double pivmin) {
  // Number of eigenvalues of T below x: sign changes of the leading principal
  // minors p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}, i.e. negative pivots
  // q_i = p_i / p_{i-1} of the LDL^T count, evaluated without divisions.  T is
  // pre-scaled to |d|, |e| <= 1, so |p| grows at most 3x per step.  The
  // sequence is renormalised by a power of two once per 8 steps, the factor
  // taken from the minors two steps before the block end and folded into the
  // next block's first two coefficients: the dependent chain is one DFMA per
  // step (an isolated zero minor counts correctly as it stands).  d / e2 are
  // padded to a multiple of 8 with d = 4, e2 = 0 (no sign change for x < 4).
  // Two consecutive zero minors (a split of T with x an eigenvalue of the
  // leading block) would stop the count: then it is redone at the next double.
  // Warps issue in order, so nothing that reads p_i may sit between its DFMA
  // and the next step's: the sign change of the pair (p_{i-2}, p_{i-1}) is
  // counted while p_i is in flight, and the next block's d / e2 are loaded
  // during the current block (measured 17 vs 36 cycles per step on one warp,
  // tools/micro/sturm_chain.cu).
  (void)pivmin;
  for (int attempt = 0; attempt < 4; ++attempt) {
    double pa = 1.0, pb = 1.0, s = 1.0;   // p_{i-2}, p_{i-1}, scale of this block
    int c = 0;
    bool dead = false;
    double nd[8], ne[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      nd[u] = d[u];
      ne[u] = (u == 0) ? 0.0 : e2[u - 1];
    }
    for (int i0 = 0; i0 < m; i0 += 8) {
      double dx[8], ee[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        dx[u] = nd[u] - x;
        ee[u] = ne[u];
      }
      {   // unconditional (no control flow around the loop-carried registers):
          // past the last block, block 0 is reloaded and not used
        const int base = (i0 + 8 < m) ? i0 + 8 : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ie = base + u - 1;
          nd[u] = d[base + u];
          const double t = e2[ie < 0 ? 0 : ie];
          ne[u] = (ie < 0) ? 0.0 : t;
        }
      }
      dx[0] *= s;
      ee[0] *= s;
      ee[1] *= s;
      double sn = 1.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double p = fma(dx[u], pb, -ee[u] * pa);
        c += (int)(((unsigned)__double2hiint(pa) ^ (unsigned)__double2hiint(pb)) >> 31);
        pa = pb;
        pb = p;
        if (u == 5) {   // 2^(-exponent of max(|p_{i0+4}|, |p_{i0+5}|)) for the next block
          const double amax = fmax(fabs(pa), fabs(pb));
          const int ex = (__double2hiint(amax) >> 20) & 0x7ff;
          sn = __hiloint2double((2046 - ex) << 20, 0);
        }
      }
      dead |= (pa == 0.0) && (pb == 0.0);
      s = sn;
    }
    c += (int)(((unsigned)__double2hiint(pa) ^ (unsigned)__double2hiint(pb)) >> 31);
    if (!dead) return c;
    x = nextafter(x, 1e300);
  }
  return 0;
}

// warp-cooperative multisection for the ascending-index-j eigenvalue of T
__device__ __forceinline__ double warp_eig_asc(const double *d, const double *e2, int m, int j, double lo, double hi,
                               double pivmin) {
  const int lane = threadIdx.x & 31;
  for (int round = 0; round < 64; ++round) {
    double tol = 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin;
    if (hi - lo <= tol) break;
    double x = fma(hi - lo, (double)(lane + 1) * (1.0 / 33.0), lo);
    int c = sturm_count(d, e2, m, x, pivmin);
    unsigned bal = __ballot_sync(0xffffffffu, c > j);
    double xlast = __shfl_sync(0xffffffffu, x, 31);
    if (bal == 0) {
      lo = xlast;
    } else {
      int f = __ffs(bal) - 1;
      double xf = __shfl_sync(0xffffffffu, x, f);
      double xp = __shfl_sync(0xffffffffu, x, f > 0 ? f - 1 : 0);
      if (f > 0) lo = xp;
      hi = xf;
    }
  }
  return 0.5 * (lo + hi);
}

// Group multisection: EG lanes per eigenvalue (EG - 1 ... split points per
// round, log2(EG + 1) bits), 32 / EG eigenvalues per warp, all groups of the
// block at once.  Computes lam[k] (descending index k in [k1, k2)) = the
// ascending-index (m - 1 - k) eigenvalue of T, scaled by bnorm.  Every lane
// derives the split points from the same (lo, hi), so no shuffles are needed.
template <int EG>
__device__ __forceinline__ void grp_multisect(const double *d, const double *e2, int m, int k1, int k2, double gl,
                                              double gu, double pivmin, double *lam, double bnorm) {
  const int lane = threadIdx.x & 31;
  const int g = lane / EG, gi = lane % EG;
  constexpr int GPW = 32 / EG;
  constexpr double STEP = 1.0 / (EG + 1);
  const int ngroups = (int)(blockDim.x >> 5) * GPW;
  const int gid = (int)(threadIdx.x >> 5) * GPW + g;
  for (int base = k1; base < k2; base += ngroups) {
    const int k = base + gid;
    const bool act = k < k2;
    const int j = m - 1 - k;
    double lo = gl, hi = gu;
    bool done = !act;
    for (int round = 0; round < 100 && __any_sync(0xffffffffu, !done); ++round) {
      // T is scaled to |d|, |e| <= 1: eigenvalues are known to ~u absolutely
      // (Householder), so an absolute floor of u / 4 loses nothing (|d sigma| <=
      // 1e-13 sigma_0 at the threshold for eps >= 1e-3).
      const double tol = 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 5.5e-17 + 2.0 * pivmin;
      if (hi - lo <= tol) done = true;
      const double x = fma(hi - lo, (double)(gi + 1) * STEP, lo);
      const int c = sturm_count(d, e2, m, x, pivmin);
      const unsigned bal = __ballot_sync(0xffffffffu, c > j);
      if (!done) {
        const unsigned gb = (EG == 32) ? bal : ((bal >> (g * EG)) & ((1u << (EG & 31)) - 1u));
        if (gb == 0) {
          lo = fma(hi - lo, (double)EG * STEP, lo);
        } else {
          const int f = __ffs(gb) - 1;
          const double xf = fma(hi - lo, (double)(f + 1) * STEP, lo);
          if (f > 0) lo = fma(hi - lo, (double)f * STEP, lo);
          hi = xf;
        }
      }
    }
    if (act && gi == 0) lam[k] = 0.5 * (lo + hi) * bnorm;
  }
}

// Inverse-iteration start vector entry (row i of vector `seed`): zero-mean,
// from a 32-bit integer hash of (row, vector).  Starts of different vectors
// must be independent, or the vectors of a cluster of (nearly) equal
// eigenvalues come out nearly parallel and their orthogonalisation amplifies
// rounding (a linear congruence whose vectors were shifted copies of one
// sequence cost up to 1e-7 of subspace accuracy on degenerate spectra).
__device__ __forceinline__ double invit_start(int i, int seed) {
  unsigned h = (unsigned)i * 0x9E3779B9u ^ ((unsigned)seed * 0x85EBCA6Bu + 0x165667B1u);
  h ^= h >> 16;
  h *= 0x7FEB352Du;
  h ^= h >> 15;
  h *= 0x846CA68Bu;
  h ^= h >> 16;
  return (double)(h >> 8) * (2.0 / 16777216.0) - 1.0;
}

// Inverse iteration for one eigenvalue lam of the tridiagonal (d, e): pivoted
// LU of T - sft I (dgttrf) then 2 solves from a fixed pseudo-random start,
// normalised.  Arrays are interleaved with stride S (S vectors side by side,
// conflict-free when S consecutive threads run S vectors); piv is one byte per
// row.  The result is written to z (contiguous, length m).
__device__ __forceinline__ void invit_one(const double *__restrict__ d, const double *__restrict__ e, int m,
                                          double sft, double pertol, int seed, double *__restrict__ DL,
                                          double *__restrict__ D, double *__restrict__ DU,
                                          double *__restrict__ DU2, double *__restrict__ b,
                                          unsigned char *__restrict__ piv, int S, double *__restrict__ z) {
  double Di = d[0] - sft, DUi = (m > 1) ? e[0] : 0.0;
#pragma unroll 2
  for (int i = 0; i < m - 1; ++i) {
    const double DLi = e[i];
    double Dn = d[i + 1] - sft;
    double DUn = (i < m - 2) ? e[i + 1] : 0.0;
    // partial pivoting by selects (threads run different vectors: no divergence)
    const bool np = fabs(Di) >= fabs(DLi);
    if (np && Di == 0.0) Di = pertol;
    const double den = np ? Di : DLi, num = np ? DLi : Di;
    const double f = num * frcp(den);
    D[i * S] = den;
    DL[i * S] = f;
    DU[i * S] = np ? DUi : Dn;
    DU2[i * S] = np ? 0.0 : DUn;
    piv[i * S] = np ? 0 : 1;
    const double nd = fma(-f, np ? DUi : Dn, np ? Dn : DUi);
    DUi = np ? DUn : -f * DUn;
    Di = nd;
  }
  D[(m - 1) * S] = Di;
#pragma unroll 4
  for (int i = 0; i < m; ++i) {  // keep pivots away from 0, store reciprocals
    double v = D[i * S];
    if (fabs(v) < pertol) v = copysign(pertol, v == 0.0 ? 1.0 : v);
    D[i * S] = frcp(v);
    b[i * S] = invit_start(i, seed);
  }
  double nrm = 0.0;
  for (int it = 0; it < 2; ++it) {
    double bi = b[0];
#pragma unroll 4
    for (int i = 0; i < m - 1; ++i) {
      const double bn = b[(i + 1) * S];
      const double l = DL[i * S];
      const bool pv = piv[i * S] != 0;
      b[i * S] = pv ? bn : bi;
      bi = fma(-l, pv ? bn : bi, pv ? bi : bn);
    }
    double x1 = bi * D[(m - 1) * S], x2 = 0.0;
    b[(m - 1) * S] = x1;
    nrm = x1 * x1;
#pragma unroll 4
    for (int i = m - 2; i >= 0; --i) {
      const double x0 = (b[i * S] - DU[i * S] * x1 - DU2[i * S] * x2) * D[i * S];
      b[i * S] = x0;
      nrm = fma(x0, x0, nrm);
      x2 = x1;
      x1 = x0;
    }
    nrm = frcp(sqrt(nrm));
    if (it < 1) {
#pragma unroll 4
      for (int i = 0; i < m; ++i) b[i * S] *= nrm;
    }
  }
#pragma unroll 4
  for (int i = 0; i < m; ++i) z[i] = b[i * S] * nrm;
}

// ------------------------------------------- one-warp eigen-solver (m <= 32) ----
// The upper levels' stacks are small (m <= 32 on the 2D configs); the block-wide
// tridiagonalisation + k_eig_t pair then spends its time in barriers and
// sequential phases sized for 512 threads.  This kernel runs the same algorithm
// (Householder tridiagonalisation, Sturm bisection, inverse iteration, MGS,
// back-transformation) in one warp per node with warp barriers only:
//   lane = row in the tridiagonalisation (G in shared memory), lane = eigenvalue
//   in the bisection, lane = vector in inverse iteration / MGS / back-transform.
// Rank by Eq. cutOff1 (or the Frobenius rule, as eig_values_phase); eps = 0
// keeps V = I, r = m (reading Z3); G = 0 gives r = 0 (Z4).
constexpr int EIGW_M = 32;
constexpr int EIGW_LD = EIGW_M + 1;
constexpr int EIGW_SMEM_DOUBLES =
    EIGW_M * EIGW_LD            /* Householder vectors (row k: v_k, v_k[k+1] = 1) */
    + 5 * 40                    /* d, e, e2 (scaled, padded to 40), tau, lam */
    + 2 * EIGW_M                /* v, w of the current step */
    + 5 * EIGW_M * EIGW_M       /* inverse-iteration LU (interleaved, stride 32) */
    + EIGW_M * EIGW_LD          /* Z: vector k at Z[k * EIGW_LD] */
    + EIGW_M * EIGW_M / 8 + 8;  /* pivot bytes */
// P Sturm counts at once (P independent recurrences interleaved: one lane's
// single count is a chain of dependent DFMAs); same arithmetic per point as
// sturm_count, a point meeting an exact zero minor is recounted by it.
template <int P>
__device__ __forceinline__ void sturm_count_multi(const double *__restrict__ d, const double *__restrict__ e2, int m,
                                                  const double (&x)[P], int (&c)[P]) {
  const double *e2m = e2 - 1;
  double p0[P], p1[P];
  bool zero[P];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    p0[q] = p1[q] = 1.0;
    c[q] = 0;
    zero[q] = false;
  }
  for (int i0 = 0; i0 < m; i0 += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      const double ee = (i == 0) ? 0.0 : e2m[i];
      const double di = d[i];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const double p2 = fma(di - x[q], p1[q], -ee * p0[q]);
        const long long b2 = __double_as_longlong(p2), b1 = __double_as_longlong(p1[q]);
        zero[q] |= (b2 << 1) == 0;
        c[q] += (int)((unsigned long long)(b2 ^ b1) >> 63);
        p0[q] = p1[q];
        p1[q] = p2;
      }
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const double a = fmax(fabs(p0[q]), fabs(p1[q]));
      const long long ex = ((__double_as_longlong(a) >> 52) & 0x7ff) - 1023;
      const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
      p0[q] *= sc;
      p1[q] *= sc;
    }
  }
#pragma unroll
  for (int q = 0; q < P; ++q)
    if (zero[q]) c[q] = sturm_count(d, e2, m, x[q], 0.0);
}

// NW warps per node: warp 0 runs every phase; with NW > 1 the eigenvalue phase
// (the longest: one lane per eigenvalue bisects ~50 Sturm counts deep) runs
// on the whole block as a group multisection with NW lanes per eigenvalue
// (log2(NW + 1) bits per round).  Waves of up to 4 nodes per SM take NW = 4,
// wider waves NW = 1 (throughput); NW = 8 is kept for the unit tests.
template <int NW>
__global__ void __launch_bounds__(32 * NW) k_eig_warp(const EigTask *__restrict__ tasks, double eps, int *status) {
  extern __shared__ double sh[];
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x];
  pdl_wait();
  const int m = t.m, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *Hv = sh, *d = Hv + EIGW_M * EIGW_LD, *e = d + 40, *e2 = e + 40, *tau = e2 + 40, *lam = tau + 40;
  double *vs = lam + 40, *ws = vs + EIGW_M, *LU = ws + EIGW_M, *Z = LU + 5 * EIGW_M * EIGW_M;
  unsigned char *pv = reinterpret_cast<unsigned char *>(Z + EIGW_M * EIGW_LD);
  if (m <= 0) {
    if (lane == 0) *t.rank_out = 0;
    return;
  }
  // row `lane` of G in registers (G symmetric: row = column); zero padding
  double g[EIGW_M];
#pragma unroll
  for (int jj = 0; jj < EIGW_M; ++jj) g[jj] = (lane < m && jj < m) ? t.G[lane + (int64_t)jj * m] : 0.0;
  double fro = 0.0, trace = 0.0;
#pragma unroll
  for (int jj = 0; jj < EIGW_M; ++jj) {
    fro = fma(g[jj], g[jj], fro);
    if (jj == lane) trace = g[jj];
  }
  fro = warp_sum(fro);
  trace = warp_sum(trace);
  if (!(fro > 0.0) || eps == 0.0) {   // G = 0: r = 0 (Z4); eps = 0: V = I, r = m (Z3)
    if (warp != 0) return;   // every warp computed the same fro: uniform exit
    const bool keep = fro > 0.0;
    if (keep)
      for (int k = 0; k < m; ++k)
        if (lane < m) t.V[lane + (int64_t)k * m] = (lane == k) ? 1.0 : 0.0;
    if (lane < m) t.sig[lane] = 0.0;
    if (lane == 0) *t.rank_out = keep ? m : 0;
    return;
  }
  if (t.dbg && threadIdx.x == 0) t.dbg[0] = clock64();
  if (warp == 0) {
  // ---- 1. Householder tridiagonalisation (lower, dsytd2), lane = row; the step
  // loop is unrolled so that every register index is static; reciprocals by
  // frcp (an IEEE FP64 division is ~430 cycles of latency on this chain) ----
#pragma unroll
  for (int k = 0; k < EIGW_M - 2; ++k) {
    if (k + 2 < m) {
      const double x = (lane > k) ? g[k] : 0.0;
      const double alpha = __shfl_sync(0xffffffffu, g[k], k + 1);
      const double s2 = warp_sum((lane > k + 1) ? x * x : 0.0);
      double tk = 0.0, beta = alpha;
      if (s2 > 0.0) {
        const double nrm2 = fma(alpha, alpha, s2), rn = frsqrt(nrm2);
        beta = -copysign(nrm2 * rn, alpha);
        tk = (beta - alpha) * frcp(beta);
        const double sc = frcp(alpha - beta);
        const double v = (lane == k + 1) ? 1.0 : ((lane > k + 1) ? x * sc : 0.0);
        vs[lane] = v;
        Hv[k * EIGW_LD + lane] = v;
        __syncwarp();
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int jj = k + 1; jj < EIGW_M; ++jj) {
          if (jj & 1) p1 = fma(g[jj], vs[jj], p1);
          else p0 = fma(g[jj], vs[jj], p0);
        }
        const double p = (lane > k) ? tk * (p0 + p1) : 0.0;
        const double a2 = -0.5 * tk * warp_sum(p * v);
        const double w = fma(a2, v, p);
        ws[lane] = w;
        __syncwarp();
        if (lane > k) {
#pragma unroll
          for (int jj = k + 1; jj < EIGW_M; ++jj) g[jj] = fma(-v, ws[jj], fma(-w, vs[jj], g[jj]));
        }
        __syncwarp();
      }
      if (lane == 0) {
        tau[k] = tk;
        e[k] = beta;
      }
    }
  }
  {
    double dl = 0.0, el = 0.0;
#pragma unroll
    for (int jj = 0; jj < EIGW_M; ++jj) {
      if (jj == lane) dl = g[jj];
      if (jj + 1 == lane) el = g[jj];
    }
    if (lane < m) d[lane] = dl;
    if (m >= 2 && lane == m - 1) e[m - 2] = el;
  }
  }   // warp 0
  if constexpr (NW > 1) __syncthreads();
  else __syncwarp();
  if (t.dbg && threadIdx.x == 0) t.dbg[1] = clock64();
  // ---- 2. eigenvalues: lane l bisects the l-th largest (Sturm counts, T / bnorm) ----
  double gl = 1e300, gu = -1e300;
  for (int i = 0; i < m; ++i) {
    const double off = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < m - 1 ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - off);
    gu = fmax(gu, d[i] + off);
  }
  const double bnorm = fmax(fmax(fabs(gl), fabs(gu)), 1e-300);
  const double isc = frcp(bnorm);
  double *ds = LU, *e2s = LU + 40;   // scaled copies (padded: d = 4, e2 = 0 beyond m)
  for (int i = threadIdx.x; i < 40; i += 32 * NW) {
    ds[i] = (i < m) ? d[i] * isc : 4.0;
    e2s[i] = (i < m - 1) ? (e[i] * isc) * (e[i] * isc) : 0.0;
  }
  double lo = gl * isc - 4.4e-16 * m - 1e-300, hi = gu * isc + 4.4e-16 * m + 1e-300;
  if constexpr (NW > 1) {
    __syncthreads();
    grp_multisect<NW>(ds, e2s, m, 0, m, lo, hi, 0.0, lam, bnorm);
    __syncthreads();
    if (warp != 0) return;
  } else {
  __syncwarp();
  const int j = m - 1 - lane;   // ascending index of this lane's eigenvalue
  {   // common bracketing: the counts at 32 points (one per lane), 33 sub-intervals
    const double h = (hi - lo) * (1.0 / 33.0);
    const int cp = sturm_count(ds, e2s, m, fma(h, (double)(lane + 1), lo), 0.0);
    int f = 32;
    for (int q = 31; q >= 0; --q)
      if (__shfl_sync(0xffffffffu, cp, q) > j) f = q;
    const double l0 = lo;
    if (f < 32) hi = fma(h, (double)(f + 1), l0);
    if (f > 0) lo = fma(h, (double)f, l0);
  }
  if (lane < m) {
    for (int it = 0; it < 200; ++it) {
      const double tol = 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 5.5e-17;
      if (hi - lo <= tol) break;
      const double mid = 0.5 * (lo + hi);
      if (sturm_count(ds, e2s, m, mid, 0.0) > j) hi = mid;
      else lo = mid;
    }
    lam[lane] = 0.5 * (lo + hi) * bnorm;
  }
  __syncwarp();
  }
  const double sig0 = sqrt(fmax(lam[0], 0.0));
  int r = 0;
  if (t.frob) {   // Eq. curOff6: smallest k with tail(k) = trace - sum_{t<k} lambda_t < budget
    const double fbud = eps * eps * (*t.frob) / t.frob_w;
    double pre = 0.0;
    while (r < m && !(trace - pre < fbud)) pre += fmax(lam[r++], 0.0);
  } else if (sig0 > 0.0) {   // lane k compares sigma_k (m <= 32)
    r = __popc(__ballot_sync(0xffffffffu, lane < m && sqrt(fmax(lam[lane], 0.0)) >= eps * sig0));
  }
  if (lane < m) t.sig[lane] = sqrt(fmax(lam[lane], 0.0));
  if (lane == 0) *t.rank_out = r;
  if (t.dbg && lane == 0) t.dbg[2] = clock64();
  if (r == 0) return;
  // ---- 3. inverse iteration, lane k < r (equal shifts separated by pertol) ----
  const double pertol = 10.0 * 2.2e-16 * bnorm;
  __syncwarp();
  if (lane < r) {
    double sft = lam[lane];
    for (int q = 1; q <= lane && lam[lane - q] - lam[lane] < pertol; ++q) sft -= pertol;
    double *DL = LU + lane, *Dv = LU + EIGW_M * EIGW_M + lane, *DU = LU + 2 * EIGW_M * EIGW_M + lane,
           *DU2 = LU + 3 * EIGW_M * EIGW_M + lane, *bb = LU + 4 * EIGW_M * EIGW_M + lane;
    invit_one(d, e, m, sft, pertol, lane, DL, Dv, DU, DU2, bb, pv + lane, EIGW_M, Z + lane * EIGW_LD);
  }
  __syncwarp();
  if (t.dbg && lane == 0) t.dbg[8] = clock64();
  // ---- 4. MGS over the r vectors (lane = vector, its elements in registers;
  // the pivot vector reaches the other lanes by shuffles) ----
  double z[EIGW_M];
#pragma unroll
  for (int i = 0; i < EIGW_M; ++i) z[i] = (lane < r && i < m) ? Z[lane * EIGW_LD + i] : 0.0;
  for (int q = 0; q < r; ++q) {
    if (lane == q) {
      double nn = 0.0;
#pragma unroll
      for (int i = 0; i < EIGW_M; ++i) nn = fma(z[i], z[i], nn);
      const double inv = nn > 0.0 ? frsqrt(nn) : 0.0;
#pragma unroll
      for (int i = 0; i < EIGW_M; ++i) z[i] *= inv;
    }
    __syncwarp();
    double zq[EIGW_M], s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < EIGW_M; ++i) {
      zq[i] = __shfl_sync(0xffffffffu, z[i], q);
      if (i & 1) s1 = fma(zq[i], z[i], s1);
      else s0 = fma(zq[i], z[i], s0);
    }
    if (lane > q && lane < r) {
      const double dt = s0 + s1;
#pragma unroll
      for (int i = 0; i < EIGW_M; ++i) z[i] = fma(-dt, zq[i], z[i]);
    }
  }
  if (t.dbg && lane == 0) t.dbg[9] = clock64();
  // ---- 5. back-transformation V = H_0 ... H_{m-3} Z (lane = vector) ----
  for (int kk = m - 3; kk >= 0; --kk) {
    const double tk = tau[kk];
    if (tk == 0.0) continue;
    const double *hv = Hv + kk * EIGW_LD;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < EIGW_M; ++i) {
      if (i & 1) s1 = fma(hv[i], z[i], s1);
      else s0 = fma(hv[i], z[i], s0);
    }
    const double sd = tk * (s0 + s1);
#pragma unroll
    for (int i = 0; i < EIGW_M; ++i) z[i] = fma(-sd, hv[i], z[i]);
  }
  if (lane < r) {
#pragma unroll
    for (int i = 0; i < EIGW_M; ++i)
      if (i < m) t.V[i + (int64_t)lane * m] = z[i];
  }
  __syncwarp();
  if (t.dbg && lane == 0) t.dbg[3] = t.dbg[4] = clock64();
  (void)status;
}

// NV simultaneous warp sums, every lane ending with all NV totals.  For NV a
// power of two: reduce-scatter (each xor stage halves the values a lane keeps)
// then one broadcast per value -- 2 NV + 4 - log2 NV exchanges instead of 5 NV
// (shuffles are a shared, low-throughput resource).  Other NV: plain butterflies.
template <int NV>
__device__ __forceinline__ void warp_sum_multi(double (&s)[NV]) {
  constexpr bool POW2 = NV > 1 && (NV & (NV - 1)) == 0 && NV <= 16;
  if constexpr (!POW2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int v = 0; v < NV; ++v) s[v] += __shfl_xor_sync(0xffffffffu, s[v], o);
  } else {
    const int lane = threadIdx.x & 31;
    double t[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) t[v] = s[v];
    int vidx = 0;   // index (0..NV-1) of the total this lane ends with
#pragma unroll
    for (int o = 16, cnt = NV; o > 0; o >>= 1) {
      if (cnt > 1) {
        const int half = cnt / 2;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < NV / 2; ++i) {
          if (i < half) {
            const double send = up ? t[i] : t[i + half];
            const double keep = up ? t[i + half] : t[i];
            t[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        if (up) vidx += half;
        cnt = half;
      } else {
        t[0] += __shfl_xor_sync(0xffffffffu, t[0], o);
      }
    }
    // broadcast: total v lives on the lanes whose stage bits spell v
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      int src = 0;
#pragma unroll
      for (int o = 16, cnt = NV, rem = v; cnt > 1; o >>= 1) {
        const int half = cnt / 2;
        if (rem >= half) {
          src |= o;
          rem -= half;
        }
        cnt = half;
      }
      s[v] = __shfl_sync(0xffffffffu, t[0], src);
    }
    (void)vidx;
  }
}

// Offset of reflector column j in the packed strictly-lower triangle (rows
// j+1..m-1 stored contiguously; index with the row i > j directly).
__device__ __forceinline__ int64_t refl_off(int j, int m) {
  return (int64_t)j * m - (int64_t)j * (j + 1) / 2 - j - 1;
}

// Back-transformation V = H_0 ... H_{m-3} Z for r columns of Z, NV columns per
// warp at once (independent reductions interleaved), Q rows per lane (m <= 32 Q).
template <int Q, int NV>
__device__ __forceinline__ void backtr_warp(double *V, const double *A, const double *tau, int m, int r,
                                            bool packed) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k0 = warp; k0 < r; k0 += nw * NV) {
    double zr[NV][Q];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int k = k0 + v * nw;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int i = lane + 32 * q;
        zr[v][q] = (k < r && i < m) ? V[(int64_t)k * m + i] : 0.0;
      }
    }
    for (int j = m - 3; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double *vj = A + (packed ? refl_off(j, m) : (int64_t)j * m);
      double vv[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int i = lane + 32 * q;
        vv[q] = (i > j && i < m) ? vj[i] : 0.0;
      }
      double s[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        s[v] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) s[v] = fma(vv[q], zr[v][q], s[v]);
      }
      warp_sum_multi<NV>(s);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double sv = s[v] * tj;
#pragma unroll
        for (int q = 0; q < Q; ++q) zr[v][q] = fma(-sv, vv[q], zr[v][q]);
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int k = k0 + v * nw;
      if (k < r)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int i = lane + 32 * q;
          if (i < m) V[(int64_t)k * m + i] = zr[v][q];
        }
    }
  }
}

// Modified Gram-Schmidt of the r inverse-iteration vectors followed by the
// back-transformation V = H_0 ... H_{m-3} Z, with the vectors held in
// registers: vector k lives in warp k % nw, slot k / nw, rows lane + 32 q.
// Per MGS step the owner warp normalises z_k and publishes it through a
// double-buffered shared vector (one block barrier per step); every warp then
// removes the z_k component from its later vectors (NV reductions interleaved).
template <int Q, int NV, bool PACKED>
__device__ __forceinline__ void orth_backtr(double *V, const double *A, const double *tau, int m, int r,
                                            double *zbuf /* 2 x 32 Q doubles of shared memory */,
                                            long long *dbg, double *stg = nullptr, int stg_cap = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double z[NV][Q];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int k = warp + v * nw;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      z[v][q] = (k < r && i < m) ? V[(int64_t)k * m + i] : 0.0;
    }
  }
  for (int k = 0; k < r; ++k) {
    double *zb = zbuf + (k & 1) * 32 * Q;
    if (warp == k % nw) {
      const int ov = k / nw;
      double zk[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        zk[q] = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (v == ov) zk[q] = z[v][q];
      }
      double s2 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) s2 = fma(zk[q], zk[q], s2);
      const double inv = frcp(sqrt(warp_sum(s2)));
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        zk[q] *= inv;
        zb[lane + 32 * q] = zk[q];
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (v == ov) z[v][q] = zk[q];
      }
    }
    __syncthreads();
    double zk[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) zk[q] = zb[lane + 32 * q];
    double s[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      s[v] = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) s[v] = fma(zk[q], z[v][q], s[v]);
    }
    warp_sum_multi<NV>(s);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int kk = warp + v * nw;
      if (kk > k && kk < r)
#pragma unroll
        for (int q = 0; q < Q; ++q) z[v][q] = fma(-s[v], zk[q], z[v][q]);
    }
  }
  if (dbg && threadIdx.x == 0) dbg[9] = clock64();
  // Reflectors in global memory (stg != nullptr): staged into shared memory in
  // chunks of ch columns (one contiguous packed segment per chunk, copied by
  // the whole block), so the per-reflector loads are shared-memory hits.
  const int ch = stg ? max(1, stg_cap / max(m, 1)) : m;
  for (int jc = m - 3; jc >= 0; jc -= ch) {
    const int jl = max(0, jc - ch + 1);
    const double *base = A;
    if (stg) {
      const int64_t lo = refl_off(jl, m) + jl + 1, hi = refl_off(jc, m) + m;
      __syncthreads();
      for (int64_t q = lo + threadIdx.x; q < hi; q += blockDim.x) stg[q - lo] = A[q];
      __syncthreads();
      base = stg - lo;
    }
  for (int j = jc; j >= jl; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    const double *vj = base + (PACKED ? refl_off(j, m) : (int64_t)j * m);
    double vv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      vv[q] = (i > j && i < m) ? vj[i] : 0.0;
    }
    double s[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      s[v] = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) s[v] = fma(vv[q], z[v][q], s[v]);
    }
    warp_sum_multi<NV>(s);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double sv = s[v] * tj;
#pragma unroll
      for (int q = 0; q < Q; ++q) z[v][q] = fma(-sv, vv[q], z[v][q]);
    }
  }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int k = warp + v * nw;
    if (k < r)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int i = lane + 32 * q;
        if (i < m) V[(int64_t)k * m + i] = z[v][q];
      }
  }
}

// Eigenvalues of the tridiagonal (d, e) for Compress (P:l.333-359, l.580-584):
// Gershgorin bounds, scaling to |T| <= 1, lambda_0 by warp multisection, the
// candidates with lambda >= (eps sigma_0)^2 / 4 by group multisection; writes
// lam[0..ncomp), t.sig, *t.rank_out; restores d; returns the rank r and the
// scale bnorm.  Every thread of the block calls it.
__device__ __forceinline__ int eig_values_phase(const EigTask &t, double eps, int m, int mp, double *d, const double *e,
                                                double *e2, double *lam, double *s_red, double *s_bc, int *s_int,
                                                double &bnorm_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // Frobenius rule: budget B = eps^2 D^2 / w on this stack's energy; tail(k) =
  // sum_{t >= k} lambda_t = trace(G) - sum_{t < k} lambda_t (the tridiagonal keeps
  // the trace); every k >= #{lambda >= B / m} has tail(k) < B, so only those
  // eigenvalues are computed
  double trace = 0.0, fbud = 0.0;
  if (t.frob) {
    double tr = 0.0;
    for (int i = tid; i < m; i += blockDim.x) tr += d[i];
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    __syncthreads();
    if (lane == 0) s_red[warp] = tr;
    __syncthreads();
    for (int w = 0; w < nw; ++w) trace += s_red[w];
    fbud = eps * eps * (*t.frob) / t.frob_w;
  }
  double gl = 1e300, gu = -1e300, emax2 = 0;
  for (int i = tid; i < m; i += blockDim.x) {
    double off = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < m - 1 ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - off);
    gu = fmax(gu, d[i] + off);
    if (i < m - 1) {
      e2[i] = e[i] * e[i];
      emax2 = fmax(emax2, e2[i]);
    }
  }
  // block min / max
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
  }
  __syncthreads();
  if (lane == 0) {
    s_red[warp] = gl;
    s_red[16 + warp] = gu;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 1e300, b = -1e300;
    for (int w = 0; w < nw; ++w) {
      a = fmin(a, s_red[w]);
      b = fmax(b, s_red[16 + w]);
    }
    s_bc[0] = a;
    s_bc[1] = b;
  }
  __syncthreads();
  if (lane == 0) s_red[warp] = emax2;
  __syncthreads();
  double em = 0;
  for (int w = 0; w < nw; ++w) em = fmax(em, s_red[w]);
  gl = s_bc[0];
  gu = s_bc[1];
  const double bnorm = fmax(fabs(gl), fabs(gu));
  // work on T / bnorm (|d|, |e| <= 1): the division-free Sturm recurrence then
  // cannot overflow within a few hundred steps; eigenvalues are scaled back.
  const double isc = 1.0 / bnorm;
  __syncthreads();
  for (int i = tid; i < mp; i += blockDim.x) {
    if (i < m) {
      d[i] *= isc;
      if (i < m - 1) e2[i] *= isc * isc;
      else e2[i] = 0.0;
    } else {
      d[i] = 4.0;   // padding: no sign change for x < 4
      e2[i] = 0.0;
    }
  }
  gl *= isc;
  gu *= isc;
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, em * isc * isc) * 1e10;
  gl -= 2.2e-16 * 2 * m + 2 * pivmin;
  gu += 2.2e-16 * 2 * m + 2 * pivmin;
  __syncthreads();
  int ncomp;
  if (m <= 64 && 4 * m <= (int)blockDim.x) {
    // small m: every eigenvalue at once (4 lanes each), no sequential lambda_0
    // pass first (for larger m computing all of them costs more than it saves)
    if (t.dbg && tid == 0) t.dbg[10] = clock64();
    ncomp = m;
    grp_multisect<4>(d, e2, m, 0, m, gl, gu, pivmin, lam, bnorm);
  } else {
    if (warp == 0) {
      double l0 = warp_eig_asc(d, e2, m, m - 1, gl, gu, pivmin);
      if (lane == 0) {
        lam[0] = l0 * bnorm;
        double thr = eps * sqrt(fmax(l0, 0.0));
        thr = 0.25 * thr * thr;
        if (t.frob) thr = fbud / m * isc;   // (scaled) candidate bound of the Frobenius rule
        int below = sturm_count(d, e2, m, thr, pivmin);
        s_int[0] = min(m, m - below + 1);  // candidates to compute (superset of kept + 1)
      }
    }
    __syncthreads();
    if (t.dbg && tid == 0) t.dbg[10] = clock64();
    ncomp = s_int[0];
    grp_multisect<4>(d, e2, m, 1, ncomp, gl, gu, pivmin, lam, bnorm);
  }
  __syncthreads();
  // restore T (inverse iteration works on the unscaled tridiagonal)
  for (int i = tid; i < m; i += blockDim.x) d[i] *= bnorm;
  __syncthreads();
  const double sig0 = sqrt(fmax(lam[0], 0.0));
  int r = 0;
  if (t.frob) {   // smallest k with tail(k) < B (Eq. curOff6)
    if (tid == 0) {
      double pre = 0.0;
      int k = 0;
      while (k < ncomp && !(trace - pre < fbud)) pre += fmax(lam[k++], 0.0);
      s_int[1] = k;
    }
    __syncthreads();
    r = s_int[1];
  } else {
    // the same comparison per candidate, one thread each (a serial loop of
    // IEEE square roots was a ~100-cycle chain link per candidate)
    for (int k0 = 0; k0 < ncomp; k0 += blockDim.x) {
      const int k = k0 + tid;
      r += __syncthreads_count(k < ncomp && sqrt(fmax(lam[k], 0.0)) >= eps * sig0);
    }
  }
  for (int k = tid; k < m; k += blockDim.x) t.sig[k] = (k < ncomp) ? sqrt(fmax(lam[k], 0.0)) : 0.0;
  if (tid == 0) *t.rank_out = r;
  bnorm_out = bnorm;
  return r;
}

// f2: squared Frobenius norm of one stored block, weighted (reading F2):
// mode 0 full block, 2 = twice the full block (SPD off-diagonal slot: both
// orientations), 1 = symmetric block from its lower triangle (SPD self slot).
struct FrobTask {
  const double *A;
  int ld, rows, cols, mode;
};
__global__ void __launch_bounds__(256) k_frob_part(const FrobTask *__restrict__ tasks, double *__restrict__ part) {
  pdl_enter();
  __shared__ double red[8];
  const FrobTask t = tasks[blockIdx.x];
  double s = 0.0;
  for (int64_t q = threadIdx.x; q < (int64_t)t.rows * t.cols; q += blockDim.x) {
    const int i = (int)(q % t.rows), j = (int)(q / t.rows);
    const double a = t.A[i + (int64_t)j * t.ld];
    if (t.mode == 1) s += (i > j) ? 2.0 * a * a : (i == j ? a * a : 0.0);
    else s += a * a;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    part[blockIdx.x] = (t.mode == 2) ? 2.0 * tot : tot;
  }
}
// *d2 += sum of part[0..n) in a fixed order (deterministic)
__global__ void __launch_bounds__(256) k_frob_final(const double *__restrict__ part, int n, double *__restrict__ d2) {
  pdl_enter();
  __shared__ double red[256];
  double s = 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x) s += part[q];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *d2 += red[0];
}

constexpr int EIG_THREADS = 256;      // generic path
constexpr int EIG_REG_THREADS = 512;  // register-tile path (m <= 128)
constexpr int EIG_REG_M = 128;
// tridiagonal record (at work + 6 m^2): d | e | tau | fro, bnorm (pad to 4m) |
// packed reflectors (m (m-1)/2) | kept eigenvalues lambda_0..lambda_{r-1}
__host__ __device__ __forceinline__ int64_t rec_lam_off(int m) { return 4 * (int64_t)m + (int64_t)m * (m - 1) / 2; }
// Householder tridiagonalisation Q^T G Q = T of one Gram matrix, m <= 128,
// with G held in registers (thread (warp w, lane) owns the 4 x 8 tile
// a[q][u] = G(32 q + lane, 8 w + u): rows strided by 32 so that the per-row
// shared-memory vectors are conflict-free).  A separate kernel so that the
// tile has the whole 128-register budget (no spills).  Output, in the task's
// global scratch at work + 6 m^2: d[128] | e[128] | tau[128] | ||G||_F^2 |
// (pad) | the packed reflectors (m (m - 1) / 2, refl_off layout), consumed by
// k_eig_t<true>.
template <bool PROF, int QR = 4, int NW = 16, int UW = 8>
__global__ void __launch_bounds__(32 * NW, 1) k_tridiag_reg(const EigTask *__restrict__ tasks, double eps,
                                                                    long long *prof) {
  constexpr int MR = 32 * QR;   // tile rows (= NW * UW columns)
  static_assert(MR == NW * UW, "square register tile");
  long long pt[6] = {0, 0, 0, 0, 0, 0}, pc = 0;
#define TRID_PROF(i)                  \
  if constexpr (PROF) {               \
    const long long tn = clock64();   \
    pt[i] += tn - pc;                 \
    pc = tn;                          \
  }
  __shared__ double s_red[32];
  __shared__ double d[MR + 8], e[MR + 8], tau[MR + 8];
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  const int m = t.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *out = t.work + 6 * (int64_t)m * m;
  double *A = out + 4 * (int64_t)m;   // packed reflectors (global)
  double a[QR][UW];
#pragma unroll
  for (int q = 0; q < QR; ++q)
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int r = 32 * q + lane, c = UW * warp + u;
      a[q][u] = (r < m && c < m) ? t.G[r + (int64_t)c * m] : 0.0;
    }
  double fro = 0;
#pragma unroll
  for (int q = 0; q < QR; ++q)
#pragma unroll
    for (int u = 0; u < UW; ++u) fro = fma(a[q][u], a[q][u], fro);
  fro = warp_sum(fro);
  if (lane == 0) s_red[warp] = fro;
  __syncthreads();
  fro = 0;
  for (int w = 0; w < NW; ++w) fro += s_red[w];
  __syncthreads();
  if (tid == 0) out[3 * m] = fro;
  if (!(fro > 0.0) || eps == 0.0) return;
  // ---- 1 (register tile). Householder tridiagonalisation, m <= 128 ----
  // A lives in registers (4 x 8 per thread, 512 threads); per step k the warp
  // owning column k forms v (written to shared memory, double-buffered, and
  // into column k of A_sm for the back-transformation), every thread forms its
  // 4 partial row sums of A v, rows reduce over the 16 column strips, and the
  // rank-2 update is register-only.  v and p vanish outside rows/cols > k, so
  // no predication is needed.  3 barriers per step.
  __shared__ double vbuf[2][MR];              // v (two buffers, 128 rows each)
  double *vsm0 = vbuf[0], *vsm1 = vbuf[1];
  __shared__ double pbuf[2][MR];              // p (two buffers)
  double *psm0 = pbuf[0], *psm1 = pbuf[1];
  // row partials of A v: static shared memory, or dynamic past 40 KB (m <= 160)
  constexpr bool DYN = NW * MR * 8 > 32 * 1024;
  __shared__ double ps_part_s[DYN ? 1 : NW][DYN ? 1 : MR];
  extern __shared__ double tr_dyn[];
  double(*ps_part)[MR] = DYN ? reinterpret_cast<double(*)[MR]>(tr_dyn) : reinterpret_cast<double(*)[MR]>(&ps_part_s[0][0]);
  __shared__ double colbuf[MR];               // column k+1 before update k
  // Householder vector of column kk from its (updated) entries col[q] = A(4 lane + q, kk),
  // run by the owner warp kk >> 3: v into the shared buffer, the packed reflector
  // store, tau and the off-diagonal beta.
  auto form_v = [&](int kk, const double *col) {
    double *vs = (kk & 1) ? vsm1 : vsm0;
    double s2 = 0;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int r = 32 * q + lane;
      if (r >= kk + 2 && r < m) s2 = fma(col[q], col[q], s2);
    }
    s2 = warp_sum(s2);
    const int rx = kk + 1;
    double x0 = 0.0;
#pragma unroll
    for (int q = 0; q < QR; ++q)
      if (32 * q + lane == rx) x0 = col[q];
    x0 = __shfl_sync(0xffffffffu, x0, rx & 31);
    double beta = x0, scal = 0.0, tk = 0.0;
    if (s2 != 0.0) {
      beta = -copysign(sqrt(fma(x0, x0, s2)), x0);
      tk = (beta - x0) * frcp(beta);
      scal = frcp(x0 - beta);
    }
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int r = 32 * q + lane;
      double v = 0.0;
      if (s2 != 0.0) v = (r == rx) ? 1.0 : ((r > rx && r < m) ? col[q] * scal : 0.0);
      vs[r] = v;
      if (r > kk && r < m) A[refl_off(kk, m) + r] = v;   // packed strictly-lower triangle
    }
    if (lane == 0) {
      tau[kk] = tk;
      e[kk] = beta;
    }
  };
  // Per step k (after the barrier that publishes v_k): partial row sums of
  // A v over the warp's 8 columns and this tile's share of v^T A v (warp
  // reduced) -> barrier -> 128 threads finish p = tau A v -> barrier -> the
  // rank-2 update A -= v w^T + w v^T (w = p + alpha v).  Look-ahead: the warp
  // owning column k+1 updates that column first and forms v_{k+1} while the
  // other warps are still updating, so the v barrier costs no extra latency.
  if (warp == 0 && m > 2) {
    double col[QR];
#pragma unroll
    for (int q = 0; q < QR; ++q) col[q] = a[q][0];
    form_v(0, col);
  }
  __syncthreads();
  if constexpr (PROF) pc = clock64();
  for (int k = 0; k < m - 2; ++k) {
    const double *vs = (k & 1) ? vsm1 : vsm0;
    double *ps = (k & 1) ? psm1 : psm0;
    const double tk = tau[k];
    // Only the trailing block changes: a warp whose 8 columns are all <= k, or
    // a row group q whose 32 rows are all <= k, multiplies / updates by exact
    // zeros (v and the masked p vanish there), so it is skipped (bitwise the
    // same result, ~1/3 of the full-tile FP64 work on average).
    const bool wact = UW * warp + UW - 1 > k;
    if (warp == ((k + 1) / UW) && k + 1 < m - 2) {
      // owner of column k+1 publishes it (as of before update k) for the form warp
      const int u1 = (k + 1) % UW;
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        double c = a[q][0];
#pragma unroll
        for (int u = 1; u < UW; ++u) c = (u1 == u) ? a[q][u] : c;
        colbuf[32 * q + lane] = c;
      }
    }
    if (wact) {
    double vc[UW];
#pragma unroll
    for (int u = 0; u < UW; ++u) vc[u] = vs[UW * warp + u];
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      if (32 * q + 31 <= k) continue;   // rows masked out of p, v_r = 0
      double s0 = 0, s1 = 0;
#pragma unroll
      for (int u = 0; u < UW; u += 2) {
        s0 = fma(a[q][u], vc[u], s0);
        if (u + 1 < UW) s1 = fma(a[q][u + 1], vc[u + 1], s1);
      }
      ps_part[warp][32 * q + lane] = s0 + s1;
    }
    } else {
#pragma unroll
      for (int q = 0; q < QR; ++q) ps_part[warp][32 * q + lane] = 0.0;
    }

    TRID_PROF(0)
    __syncthreads();                                              // (2) partials visible
    TRID_PROF(1)
    if (tid < MR) {
      double sacc;
      if constexpr (QR >= 5) {   // larger tile: four running sums (fewer live registers)
        double h4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int w = 0; w < NW; ++w) h4[w & 3] += ps_part[w][tid];
        sacc = (h4[0] + h4[1]) + (h4[2] + h4[3]);
      } else {
      double h[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) h[w] = ps_part[w][tid];
      constexpr int P2 = (NW >= 32) ? 32 : (NW >= 16) ? 16 : (NW >= 8) ? 8 : (NW >= 4) ? 4 : (NW >= 2) ? 2 : 1;
#pragma unroll
      for (int w = P2; w < NW; ++w) h[w - P2] += h[w];      // NW not a power of two
#pragma unroll
      for (int st = P2 / 2; st > 0; st /= 2)
#pragma unroll
        for (int w = 0; w < st; ++w) h[w] += h[w + st];   // pairwise tree
      sacc = h[0];
      }
      const double pi = (tid > k && tid < m) ? tk * sacc : 0.0;
      ps[tid] = pi;
      // p.v over the 128 rows: 4 warp reductions (shuffles are a shared,
      // low-throughput resource; 16 warps reducing would cost ~4x more)
      const double pvw = warp_sum(pi * vs[tid]);
      if (lane == 0) s_red[warp] = pvw;
    }
    TRID_PROF(2)
    __syncthreads();                                              // (3) p visible
    TRID_PROF(3)
    double pv;
    if constexpr (QR == 4) pv = (s_red[0] + s_red[1]) + (s_red[2] + s_red[3]);
    else if constexpr (QR == 2) pv = s_red[0] + s_red[1];
    else if constexpr (QR == 1) pv = s_red[0];
    else {
      pv = s_red[0];
#pragma unroll
      for (int w = 1; w < QR; ++w) pv += s_red[w];
    }
    const double alpha = -0.5 * tk * pv;
    // (vr, wr, v_c, w_c are re-read from shared memory here: with the 32-double
    // tile live, keeping them in registers across form_v would spill)
    const double *psc = ps + UW * warp, *vsc = vs + UW * warp;
    if (wact && QR <= 4) {
      double vq[QR], wq[QR];
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        vq[q] = vs[32 * q + lane];
        wq[q] = fma(alpha, vq[q], ps[32 * q + lane]);
      }
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const double vcu = vsc[u], wcu = fma(alpha, vcu, psc[u]);
#pragma unroll
        for (int q = 0; q < QR; ++q)
          if (32 * q + 31 > k) a[q][u] = fma(-vq[q], wcu, fma(-wq[q], vcu, a[q][u]));
      }
    } else if (wact) {   // larger tile: row-outer, the column values re-read (fewer live registers)
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        if (32 * q + 31 <= k) continue;
        const double vq = vs[32 * q + lane], wq = fma(alpha, vq, ps[32 * q + lane]);
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          const double vcu = vsc[u], wcu = fma(alpha, vcu, psc[u]);
          a[q][u] = fma(-vq, wcu, fma(-wq, vcu, a[q][u]));
        }
      }
    }
    const int k1 = k + 1;
    // v_{k+1} is formed by a warp whose own columns are finished (warp 0 once
    // k >= 7; warp 15 before), from the published column and the same update
    // formula the owner applies in registers (bitwise the same column), so it
    // overlaps the other warps' updates instead of trailing the owner's.
    if (warp == (k1 >= UW ? 0 : NW - 1) && k1 < m - 2) {
      const double vcu = vs[k1], wcu = fma(alpha, vcu, ps[k1]);
      double col[QR];
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        const double vq = vs[32 * q + lane], wq = fma(alpha, vq, ps[32 * q + lane]);
        col[q] = fma(-vq, wcu, fma(-wq, vcu, colbuf[32 * q + lane]));
      }
      form_v(k1, col);
    }
    TRID_PROF(4)
    __syncthreads();                                              // (1) v_{k+1} visible
    TRID_PROF(5)
  }
  if constexpr (PROF) {
    if (lane == 0)
      for (int i = 0; i < 6; ++i) prof[warp * 8 + i] = pt[i];
  }
#undef TRID_PROF
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
  for (int i = tid; i < m; i += blockDim.x) {
    out[i] = d[i];
    out[m + i] = e[i];
    out[2 * m + i] = tau[i];
  }
}


// DSMEM helpers: shared::cluster address of `p` in CTA `rank` of the cluster,
// and 64-bit loads / stores through it (no generic-address window checks).
__device__ __forceinline__ uint32_t dsm_addr(const void *p, int rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double dsm_ld(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void dsm_st(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// ------------------------------------------- cluster tridiagonalisation ----
// Householder tridiagonalisation of one Gram matrix with 128 < m <= 32 QR,
// spread over a thread-block cluster of CL CTAs (distributed shared memory):
// CTA j holds the column strip [16 UC j, 16 UC (j+1)) in registers (thread
// (warp w, lane) owns a[q][u] = G(32 q + lane, 16 UC j + UC w + u)).  Per
// step k:
//   A  every active warp forms p_c = (A v_k)_c for its UC columns as column
//      dots (A symmetric), rows over the lanes, finished 32-row tiles skipped,
//      and writes them to the L2 exchange (the strips partition the columns,
//      so p is gathered, not summed); the owner warp of column k+1 publishes
//      that column;
//   C  cluster barrier; p_t = tau_k (A v)_t read by every CTA, masked to t > k;
//      p.v reduced in the same order everywhere;
//   D  rank-2 update of the strip;
//   E  every CTA applies update k to the published column k+1 and forms
//      v_{k+1} and tau_{k+1} itself (the same arithmetic on the same data in
//      every CTA, so bitwise the same); one cluster barrier per step.
// Output in the same tridiagonal record as k_tridiag_reg.
// Dynamic shared memory: 21 * 32 QR doubles.
template <int QR, int UC, int CL>
__global__ void __launch_bounds__(512, 1) k_tridiag_cl(const EigTask *__restrict__ tasks, double eps,
                                                       long long *prof = nullptr) {
  long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pc = 0;
#define TCL_PROF(i)                                  \
  if (prof && threadIdx.x == 0 && blockIdx.x == 0) { \
    const long long tn = clock64();                  \
    pt[i] += tn - pc;                                \
    pc = tn;                                         \
  }
  constexpr int MMAX = 32 * QR;
  constexpr int CW = 16 * UC;   // columns per CTA
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  // dynamic shared memory: vbuf[2][MMAX] | (unused 16 MMAX) | pcta | psm | colbuf
  extern __shared__ double dsh[];
  double(*vbuf)[MMAX] = reinterpret_cast<double(*)[MMAX]>(dsh);
  double *pcta = dsh + 18 * MMAX, *psm = dsh + 19 * MMAX, *colbuf = dsh + 20 * MMAX;
  __shared__ double taub[2];
  __shared__ double s_red[16];
  __shared__ double s_fro[CL];
  const EigTask t = tasks[blockIdx.x / CL];
  const int m = t.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = rank * CW + warp * UC;   // first column of this warp
  double *out = t.work + 6 * (int64_t)m * m;
  double *A = out + 4 * (int64_t)m;        // packed reflectors (global)
  // Exchanges go through L2 (global scratch at work[0..), free in this path):
  // DSMEM serves ~1 thread-request per cycle per SM, too slow for the
  // all-gather of CL partial vectors; coalesced L2 traffic is not.
  double *xg = t.work;                                  // [2][MMAX] p = A v (all-gather)
  double *vg = t.work + 2 * CL * MMAX;                  // [2][MMAX + 8] v and tau
  double a[QR][UC];
#pragma unroll
  for (int q = 0; q < QR; ++q)
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const int r = 32 * q + lane, c = c0 + u;
      a[q][u] = (r < m && c < m) ? t.G[r + (int64_t)c * m] : 0.0;
    }
  // ||G||_F^2: CTA partial pushed to every CTA, summed in rank order
  {
    double f = 0;
#pragma unroll
    for (int q = 0; q < QR; ++q)
#pragma unroll
      for (int u = 0; u < UC; ++u) f = fma(a[q][u], a[q][u], f);
    f = warp_sum(f);
    if (lane == 0) s_red[warp] = f;
    __syncthreads();
    if (tid < CL) {
      double fc = 0;
      for (int w = 0; w < 16; ++w) fc += s_red[w];
      *cl.map_shared_rank(&s_fro[rank], tid) = fc;
    }
    cl.sync();
  }
  double fro = 0;
  for (int j = 0; j < CL; ++j) fro += s_fro[j];
  if (rank == 0 && tid == 0) out[3 * m] = fro;
  if (!(fro > 0.0) || eps == 0.0) return;   // uniform over the cluster

  // v of column kk from its updated entries col[q] (rows 32 q + lane), by one
  // warp: pushed (with tau) into every CTA of the cluster; e, tau and the
  // packed reflector to the global record.
  auto form_v = [&](int kk, const double *col) {
    double s2 = 0;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int r = 32 * q + lane;
      if (r >= kk + 2 && r < m) s2 = fma(col[q], col[q], s2);
    }
    s2 = warp_sum(s2);
    const int rx = kk + 1;
    double x0 = 0.0;
#pragma unroll
    for (int q = 0; q < QR; ++q)
      if (32 * q + lane == rx) x0 = col[q];
    x0 = __shfl_sync(0xffffffffu, x0, rx & 31);
    double beta = x0, scal = 0.0, tk = 0.0;
    if (s2 != 0.0) {
      beta = -copysign(sqrt(fma(x0, x0, s2)), x0);
      tk = (beta - x0) * frcp(beta);
      scal = frcp(x0 - beta);
    }
    const int b = kk & 1;
#pragma unroll
    for (int q = 0; q < QR; ++q) {
      const int r = 32 * q + lane;
      double v = 0.0;
      if (s2 != 0.0) v = (r == rx) ? 1.0 : ((r > rx && r < m) ? col[q] * scal : 0.0);
      vg[b * (MMAX + 8) + r] = v;   // every CTA reads it after the cluster barrier
      if (r > kk && r < m) A[refl_off(kk, m) + r] = v;
    }
    if (lane == 0) vg[b * (MMAX + 8) + MMAX] = tk;
    if (lane == 0) {
      out[2 * m + kk] = tk;
      out[m + kk] = beta;
    }
  };
  // v_0: column 0 lives in CTA 0, warp 0, u = 0
  // every CTA copies v_kk (and tau) from the CTA that formed it (pull: one
  // remote load per thread instead of QR x CL serial remote stores in one warp)
  auto pull_v = [&](int kk) {
    const int b = kk & 1;
    for (int r = tid; r < MMAX; r += blockDim.x) vbuf[b][r] = __ldcg(vg + b * (MMAX + 8) + r);
    if (tid == 0) taub[b] = __ldcg(vg + b * (MMAX + 8) + MMAX);
    __syncthreads();
  };
  if (rank == 0 && warp == 0 && m > 2) {
    double col[QR];
#pragma unroll
    for (int q = 0; q < QR; ++q) col[q] = a[q][0];
    form_v(0, col);
  }
  cl.sync();
  if (m > 2) pull_v(0);
  // column k+1 as of A_k, published by its owner warp with the partials: every
  // CTA then applies update k to it and forms v_{k+1} itself (the same
  // arithmetic on the same data in every CTA, so bitwise the same v), which
  // leaves one cluster barrier per step instead of two plus a pull of v
  double *colg = vg + 2 * (MMAX + 8);    // [2][MMAX] published column
  double *colp = pcta;                   // updated column k+1 (shared)
  __shared__ double s_red2[16];
  if (prof && threadIdx.x == 0 && blockIdx.x == 0) pc = clock64();
  for (int k = 0; k < m - 2; ++k) {
    const double *vs = vbuf[k & 1];
    const double tk = taub[k & 1];
    const int k1 = k + 1;
    const bool own1 = k1 < m - 2 && k1 >= rank * CW && k1 < (rank + 1) * CW;   // column k+1 is ours
    // ---- A ----
    if (own1 && warp == (k1 - rank * CW) / UC) {
      const int u1 = (k1 - rank * CW) % UC;
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        double c = a[q][0];
#pragma unroll
        for (int u = 1; u < UC; ++u) c = (u1 == u) ? a[q][u] : c;
        colg[(k & 1) * MMAX + 32 * q + lane] = c;
      }
    }
    const bool wact = c0 + UC - 1 > k;
    if (wact) {
      // (A v)_c for the warp's columns c as column dots (A symmetric: column c
      // = row c), rows over the lanes: no cross-warp partials to combine, the
      // cluster exchanges the MMAX entries of p once (all-gather through L2)
      double s[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) s[u] = 0.0;
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        if (32 * q + 31 <= k) continue;
        const double vr = vs[32 * q + lane];
#pragma unroll
        for (int u = 0; u < UC; ++u) s[u] = fma(a[q][u], vr, s[u]);
      }
      warp_sum_multi<UC>(s);
      double pl = s[0];
#pragma unroll
      for (int u = 1; u < UC; ++u) pl = (lane == u) ? s[u] : pl;
      if (lane < UC) xg[(k & 1) * MMAX + c0 + lane] = pl;
    }
    TCL_PROF(0)
    TCL_PROF(1)
    TCL_PROF(2)
    cl.sync();
    TCL_PROF(3)
    // ---- C ----
    double colr = 0.0;   // column k+1 (as of A_k), row tid
    if (tid < MMAX) {
      const double sacc = __ldcg(xg + (k & 1) * MMAX + tid);
      if (k1 < m - 2) colr = __ldcg(colg + (k & 1) * MMAX + tid);
      const double pi = (tid > k && tid < m) ? tk * sacc : 0.0;
      psm[tid] = pi;
      const double pvw = warp_sum(pi * vs[tid]);
      if (lane == 0) s_red[warp] = pvw;
    }
    TCL_PROF(4)
    __syncthreads();
    double pv = 0.0;
#pragma unroll
    for (int w = 0; w < MMAX / 32; ++w) pv += s_red[w];
    const double alpha = -0.5 * tk * pv;
    // ---- D ----
    if (wact) {
      double vq[QR], wq[QR];
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        vq[q] = vs[32 * q + lane];
        wq[q] = fma(alpha, vq[q], psm[32 * q + lane]);
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int c = c0 + u;
        const double vcu = (c < MMAX) ? vs[c] : 0.0, wcu = fma(alpha, vcu, (c < MMAX) ? psm[c] : 0.0);
#pragma unroll
        for (int q = 0; q < QR; ++q)
          if (32 * q + 31 > k) a[q][u] = fma(-vq[q], wcu, fma(-wq[q], vcu, a[q][u]));
      }
    }
    TCL_PROF(5)
    // ---- E: v_{k+1} in every CTA ----
    if (k1 < m - 2) {
      const double vcu = vs[k1], wcu = fma(alpha, vcu, psm[k1]);
      double s2p = 0.0;
      if (tid < MMAX) {
        const double vq = vs[tid], wq = fma(alpha, vq, psm[tid]);
        const double cu = fma(-vq, wcu, fma(-wq, vcu, colr));
        colp[tid] = cu;
        if (tid >= k1 + 2 && tid < m) s2p = cu * cu;
      }
      s2p = warp_sum(s2p);
      if (lane == 0) s_red2[warp] = s2p;
      __syncthreads();
      double s2 = 0.0;
#pragma unroll
      for (int w = 0; w < MMAX / 32; ++w) s2 += s_red2[w];
      const int rx = k1 + 1;
      const double x0 = colp[rx];
      double beta = x0, scal = 0.0, tk1 = 0.0;
      if (s2 != 0.0) {
        const double nrm2 = fma(x0, x0, s2);
        beta = -copysign(nrm2 * frsqrt(nrm2), x0);
        tk1 = (beta - x0) * frcp(beta);
        scal = frcp(x0 - beta);
      }
      const int b = k1 & 1;
      if (tid < MMAX) {
        const int r = tid;
        double v = 0.0;
        if (s2 != 0.0) v = (r == rx) ? 1.0 : ((r > rx && r < m) ? colp[r] * scal : 0.0);
        vbuf[b][r] = v;
        if (rank == 0 && r > k1 && r < m) A[refl_off(k1, m) + r] = v;
      }
      if (tid == 0) {
        taub[b] = tk1;
        if (rank == 0) {
          out[2 * m + k1] = tk1;
          out[m + k1] = beta;
        }
      }
      __syncthreads();
    }
    TCL_PROF(6)
  }
  if (prof && threadIdx.x == 0 && blockIdx.x == 0)
    for (int q = 0; q < 8; ++q) prof[q] = pt[q];
#undef TCL_PROF
  // diagonal and the last sub-diagonal from the register tiles
#pragma unroll
  for (int q = 0; q < QR; ++q)
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const int r = 32 * q + lane, c = c0 + u;
      if (r < m && r == c) out[r] = a[q][u];
      if (m >= 2 && r == m - 1 && c == m - 2) out[m + m - 2] = a[q][u];
    }
  if (rank == 0 && tid == 0) {
    out[m + m - 1] = 0.0;
    if (m >= 2) out[2 * m + m - 2] = 0.0;
    out[2 * m + m - 1] = 0.0;
  }
}

// REG: tridiagonal record from k_tridiag_reg (m <= 128, reflectors copied to
// shared memory); PRE: record from k_tridiag_cl (128 < m <= 512, reflectors
// read from the global record); neither: tridiagonalise here (generic path).
template <bool REG, bool PRE = false>
__global__ void __launch_bounds__((REG || PRE) ? EIG_REG_THREADS : EIG_THREADS)
    k_eig_t(const EigTask *__restrict__ tasks, double eps, int smem_cap_doubles, int *status) {
  extern __shared__ double sh[];
  __shared__ double s_red[32];
  __shared__ double s_bc[8];
  __shared__ int s_int[4];
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  const int m = t.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int ml = m > 512 ? m : 512;  // lam doubles as p-partials scratch during phase 1
  const int mp = (m + 8) & ~7;       // padded length (>= m + 1, multiple of 8)
  double *d = sh, *e = d + mp, *tau = e + mp, *e2 = tau + mp, *vt = e2 + mp, *pw = vt + mp, *lam = pw + mp;
  double *A = PRE ? t.work + 6 * (int64_t)m * m + 4 * (int64_t)m
                 : ((REG || (int64_t)m * m + 6 * mp + ml <= smem_cap_doubles) ? lam + ml
                                                                              : t.work + 6 * (int64_t)m * m);
  double *scr = t.work;  // 6 m^2: inverse-iteration scratch
  if constexpr (!REG && !PRE) {
    for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x) A[q] = t.G[q];
    __syncthreads();
  }
  if (t.dbg && tid == 0) t.dbg[0] = clock64();
  // block reduction helper (sum)
  auto bsum = [&](double v) -> double {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double r = 0;
    for (int w = 0; w < nw; ++w) r += s_red[w];
    return r;
  };
  double fro = 0;
  if constexpr (REG || PRE) {
    fro = t.work[6 * (int64_t)m * m + 3 * m];   // ||G||_F^2 from the tridiagonal record
  } else {
    for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x) fro += A[q] * A[q];
    fro = bsum(fro);
  }
  if (!(fro > 0.0)) {
    if (tid == 0) *t.rank_out = 0;
    for (int q = tid; q < m; q += blockDim.x) t.sig[q] = 0.0;
    return;
  }
  if (eps == 0.0) {
    for (int64_t q = tid; q < (int64_t)m * m; q += blockDim.x) t.V[q] = ((q % m) == (q / m)) ? 1.0 : 0.0;
    for (int q = tid; q < m; q += blockDim.x) t.sig[q] = 0.0;
    if (tid == 0) *t.rank_out = m;
    return;
  }
  if constexpr (REG || PRE) {
  // ---- 1: done by k_tridiag_reg / k_tridiag_cl; load T (and, REG, the reflectors) ----
  {
    const double *in = t.work + 6 * (int64_t)m * m;
    for (int i = tid; i < m; i += blockDim.x) {
      d[i] = in[i];
      e[i] = in[m + i];
      tau[i] = in[2 * m + i];
    }
    if constexpr (REG) {
      const int64_t np = (int64_t)m * (m - 1) / 2;
      for (int64_t q = tid; q < np; q += blockDim.x) A[q] = in[4 * (int64_t)m + q];
    }
    __syncthreads();
  }
  } else {
  // ---- 1. Householder tridiagonalisation (thread per row) ----
  // step k: v from column k (its squared norm below x0 comes from the previous
  // step), p = tau A22 v (thread i owns row i: sum over columns, conflict-free
  // shared-memory reads), alpha from p.v, A22 -= v w^T + w v^T with
  // w = p + alpha v formed on the fly, and the next column's norm; 3 barriers.
  __shared__ double s_red2[32];
  {
    double a = 0;
    for (int i = 2 + tid; i < m; i += blockDim.x) a = fma(A[i], A[i], a);
    a = warp_sum(a);
    if (lane == 0) s_red2[warp] = a;
    __syncthreads();
  }
  long long tph[4] = {0, 0, 0, 0};
  long long tprev = clock64();
  for (int k = 0; k < m - 2; ++k) {
    const int L = m - k - 1;
    double *colk = A + (int64_t)k * m + (k + 1);   // x = A[k+1.., k], length L
    double *A22 = A + (int64_t)(k + 1) * m + (k + 1);
    double s2 = 0;                      // squared norm below x0 (partials of the last step)
    for (int w = 0; w < nw; ++w) s2 += s_red2[w];
    const double x0 = colk[0];
    double beta = x0, tk = 0.0, scal = 0.0;
    const bool refl = s2 != 0.0;
    if (refl) {
      beta = -copysign(sqrt(x0 * x0 + s2), x0);
      tk = (beta - x0) * frcp(beta);
      scal = frcp(x0 - beta);
      for (int i = tid; i < L; i += blockDim.x) {
        const double v = (i == 0) ? 1.0 : colk[i] * scal;
        vt[i] = v;
        colk[i] = v;
      }
    }
    if (tid == 0) {
      tau[k] = tk;
      e[k] = beta;
    }
    __syncthreads();                                              // (1) v visible
    if (t.dbg && tid == 0) { long long tn = clock64(); tph[0] += tn - tprev; tprev = tn; }
    double pvp = 0;
    if (refl) {
      for (int i = tid; i < L; i += blockDim.x) {
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int j = 0;
        for (; j + 3 < L; j += 4) {
          a0 = fma(A22[i + (int64_t)j * m], vt[j], a0);
          a1 = fma(A22[i + (int64_t)(j + 1) * m], vt[j + 1], a1);
          a2 = fma(A22[i + (int64_t)(j + 2) * m], vt[j + 2], a2);
          a3 = fma(A22[i + (int64_t)(j + 3) * m], vt[j + 3], a3);
        }
        for (; j < L; ++j) a0 = fma(A22[i + (int64_t)j * m], vt[j], a0);
        const double pi = tk * ((a0 + a1) + (a2 + a3));
        pw[i] = pi;
        pvp = fma(pi, vt[i], pvp);
      }
    }
    pvp = warp_sum(pvp);
    if (lane == 0) s_red[warp] = pvp;
    __syncthreads();                                              // (2) p, partials visible
    if (t.dbg && tid == 0) { long long tn = clock64(); tph[1] += tn - tprev; tprev = tn; }
    double nxt = 0;
    if (refl) {
      double pv = 0;
      for (int w = 0; w < nw; ++w) pv += s_red[w];
      const double alpha = -0.5 * tk * pv;
      for (int i = tid; i < L; i += blockDim.x) {
        const double vi = vt[i], wi = fma(alpha, vi, pw[i]);
        int j = 0;
        for (; j + 1 < L; j += 2) {
          const double vj0 = vt[j], wj0 = fma(alpha, vj0, pw[j]);
          const double vj1 = vt[j + 1], wj1 = fma(alpha, vj1, pw[j + 1]);
          double *c0 = A22 + i + (int64_t)j * m, *c1 = c0 + m;
          *c0 -= fma(vi, wj0, wi * vj0);
          *c1 -= fma(vi, wj1, wi * vj1);
        }
        if (j < L) {
          const double vj0 = vt[j], wj0 = fma(alpha, vj0, pw[j]);
          A22[i + (int64_t)j * m] -= fma(vi, wj0, wi * vj0);
        }
        if (i >= 2) nxt = fma(A22[i], A22[i], nxt);   // column 0 of A22 = next column
      }
    } else {
      for (int i = 2 + tid; i < L; i += blockDim.x) nxt = fma(A22[i], A22[i], nxt);
    }
    nxt = warp_sum(nxt);
    if (lane == 0) s_red2[warp] = nxt;   // read by every thread at the next step's start
    __syncthreads();                                              // (3) A22, partials
    if (t.dbg && tid == 0) { long long tn = clock64(); tph[2] += tn - tprev; tprev = tn; }
  }
  if (t.dbg && tid == 0) for (int q = 0; q < 3; ++q) t.dbg[5 + q] = tph[q];
  for (int i = tid; i < m; i += blockDim.x) d[i] = A[i + (int64_t)i * m];
  if (tid == 0) {
    if (m >= 2) e[m - 2] = A[(m - 1) + (int64_t)(m - 2) * m];
    e[m - 1] = 0.0;
    if (m >= 2) tau[m - 2] = 0.0;
    tau[m - 1] = 0.0;
  }
  __syncthreads();
  }
  if (t.dbg && tid == 0) t.dbg[1] = clock64();
  // ---- 2. eigenvalues (Sturm multisection) ----
  double bnorm;
  const int r = eig_values_phase(t, eps, m, mp, d, e, e2, lam, s_red, s_bc, s_int, bnorm);
  if constexpr (PRE) {
    // PRE pipeline stage 0 ends here: the kept eigenvalues and ||T|| bound go to
    // the tridiagonal record for k_invit_multi; MGS + back-transformation follow
    // in k_orth_bgs / k_backtr_multi.
    double *rec = t.work + 6 * (int64_t)m * m;
    for (int k = tid; k < r; k += blockDim.x) rec[rec_lam_off(m) + k] = lam[k];
    if (tid == 0) rec[3 * m + 1] = bnorm;
    return;
  }
  if (t.dbg && tid == 0) t.dbg[2] = clock64();
  // ---- 4. inverse iteration, one thread per kept eigenvalue ----
  // Each vector is computed independently (shift lambda_k, equal shifts
  // separated by pertol), then the r vectors are orthonormalised (MGS): mixing
  // kept vectors leaves the kept subspace unchanged.
  const double pertol = 10.0 * 2.2e-16 * bnorm;
  const bool a_in_smem = !PRE && (REG || (int64_t)m * m + 6 * mp + ml <= smem_cap_doubles);
  const int64_t used = 6 * (int64_t)mp + ml + (REG ? (int64_t)m * (m - 1) / 2 : (a_in_smem ? (int64_t)m * m : 0));
  const int64_t per = 5 * (int64_t)m + (m + 7) / 8;   // doubles per vector (5 arrays + piv bytes)
  const int64_t avail = (int64_t)smem_cap_doubles - used;
  if (avail >= per) {
    // batches of nbv vectors with their LU / right-hand side in shared memory
    const int nbv = (int)min(min(avail / per, (int64_t)r), (int64_t)blockDim.x);
    double *ws = sh + used;
    for (int k0 = 0; k0 < r; k0 += nbv) {
      const int nb = min(nbv, r - k0);
      const int kk = tid;
      if (kk < nb) {
        const int k = k0 + kk;
        double sft = lam[k];
        for (int q = 1; q <= k && lam[k - q] - lam[k] < pertol; ++q) sft -= pertol;
        double *DL = ws + kk, *Dv = DL + (int64_t)m * nb, *DU = Dv + (int64_t)m * nb, *DU2 = DU + (int64_t)m * nb,
               *bb = DU2 + (int64_t)m * nb;
        unsigned char *pv = reinterpret_cast<unsigned char *>(ws + 5 * (int64_t)m * nb) + kk;
        invit_one(d, e, m, sft, pertol, k, DL, Dv, DU, DU2, bb, pv, nb, t.V + (int64_t)k * m);
      }
      __syncthreads();
    }
  } else
  for (int k = tid; k < r; k += blockDim.x) {
    // interleaved scratch: element i of vector k at [i * r + k] (coalesced across threads)
    const int64_t RR = r;
    double *DL = scr + k, *D = DL + m * RR, *DU = D + m * RR, *DU2 = DU + m * RR, *b = DU2 + m * RR,
           *piv = b + m * RR;
    double sft = lam[k];
    for (int q = 1; q <= k && lam[k - q] - lam[k] < pertol; ++q) sft -= pertol;
    // dgttrf on T - sft I with the running pivot row carried in registers
    double Di = d[0] - sft, DUi = (m > 1) ? e[0] : 0.0;
#pragma unroll 2
    for (int i = 0; i < m - 1; ++i) {
      const double DLi = e[i];
      double Dn = d[i + 1] - sft;
      double DUn = (i < m - 2) ? e[i + 1] : 0.0;
      if (fabs(Di) >= fabs(DLi)) {
        if (Di == 0.0) Di = pertol;
        const double f = DLi * frcp(Di);
        D[(i) * RR] = Di;
        DL[(i) * RR] = f;
        DU[(i) * RR] = DUi;
        DU2[(i) * RR] = 0.0;
        piv[(i) * RR] = 0.0;
        Dn = fma(-f, DUi, Dn);
      } else {
        const double f = Di * frcp(DLi);
        D[(i) * RR] = DLi;
        DL[(i) * RR] = f;
        DU[(i) * RR] = Dn;
        DU2[(i) * RR] = DUn;
        piv[(i) * RR] = 1.0;
        const double nd = fma(-f, Dn, DUi);
        DUn = -f * DUn;
        Dn = nd;
      }
      Di = Dn;
      DUi = DUn;
    }
    D[(m - 1) * RR] = Di;
    for (int i = 0; i < m; ++i) {        // keep pivots away from 0, store reciprocals
      double v = D[(i) * RR];
      if (fabs(v) < pertol) v = copysign(pertol, v == 0.0 ? 1.0 : v);
      D[(i) * RR] = frcp(v);
    }
    for (int i = 0; i < m; ++i) b[(i) * RR] = invit_start(i, k);
    for (int it = 0; it < 3; ++it) {
      // forward (row interchanges + unit lower)
      double bi = b[(0) * RR];
#pragma unroll 4
      for (int i = 0; i < m - 1; ++i) {
        const double bn = b[(i + 1) * RR];
        if (piv[(i) * RR] == 0.0) {
          b[(i) * RR] = bi;
          bi = fma(-DL[(i) * RR], bi, bn);
        } else {
          b[(i) * RR] = bn;
          bi = fma(-DL[(i) * RR], bn, bi);
        }
      }
      b[(m - 1) * RR] = bi;
      // backward (upper with two super-diagonals), carries x_{i+1}, x_{i+2}
      double x1 = b[(m - 1) * RR] * D[(m - 1) * RR];
      b[(m - 1) * RR] = x1;
      double nrm = x1 * x1, x2 = 0.0;
      if (m >= 2) {
        const double x0 = (b[(m - 2) * RR] - DU[(m - 2) * RR] * x1) * D[(m - 2) * RR];
        b[(m - 2) * RR] = x0;
        nrm = fma(x0, x0, nrm);
        x2 = x1;
        x1 = x0;
      }
#pragma unroll 4
      for (int i = m - 3; i >= 0; --i) {
        const double x0 = (b[(i) * RR] - DU[(i) * RR] * x1 - DU2[(i) * RR] * x2) * D[(i) * RR];
        b[(i) * RR] = x0;
        nrm = fma(x0, x0, nrm);
        x2 = x1;
        x1 = x0;
      }
      nrm = frcp(sqrt(nrm));
      for (int i = 0; i < m; ++i) b[(i) * RR] *= nrm;
    }
    double *z = t.V + (int64_t)k * m;
    for (int i = 0; i < m; ++i) z[i] = b[(i) * RR];
  }
  __syncthreads();
  // ---- 4b/5. orthonormalisation + back-transformation V = H_0 ... H_{m-3} Z ----
  {
    if (t.dbg && tid == 0) t.dbg[8] = clock64();
    double *s_zb = lam;   // eigenvalues are no longer needed (2 x 32 Q <= 512 doubles)
    const int per_w = (r + nw - 1) / nw;
    if constexpr (PRE) {
      // register-resident vectors, 16 warps, packed reflectors in global memory
      double *zb = sh + 6 * (int64_t)mp + ml;   // inverse-iteration workspace (free now)
      const int stg_cap = smem_cap_doubles - (6 * mp + ml) - 1024;   // reflector staging
      bool done = true;
      if (m <= 256 && per_w <= 4) {
        if (per_w > 2) orth_backtr<8, 4, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
        else if (per_w > 1) orth_backtr<8, 2, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
        else orth_backtr<8, 1, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
      } else if (m <= 384 && per_w <= 3) {
        if (per_w > 2) orth_backtr<12, 3, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
        else if (per_w > 1) orth_backtr<12, 2, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
        else orth_backtr<12, 1, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
      } else if (m <= 512 && per_w <= 2) {
        if (per_w > 1) orth_backtr<16, 2, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
        else orth_backtr<16, 1, true>(t.V, A, tau, m, r, zb, t.dbg, zb + 1024, stg_cap);
      } else {
        done = false;
      }
      if (done) {
        __syncthreads();
        if (t.dbg && tid == 0) t.dbg[3] = t.dbg[4] = clock64();
        return;
      }
    } else if (REG || m <= 64) {
      // register-resident vectors (REG: m <= 128, 16 warps; generic: m <= 64, 8 warps)
      if (REG) {
        if (per_w > 8) {   // 8-warp launch with r > 64 (only from a wrong rank prediction)
          if (tid == 0 && atomicCAS(&status[0], 0, -4) == 0) status[1] = t.node;
          return;
        }
        if (per_w > 4) orth_backtr<4, 8, true>(t.V, A, tau, m, r, s_zb, t.dbg);
        else if (per_w > 2) orth_backtr<4, 4, true>(t.V, A, tau, m, r, s_zb, t.dbg);
        else if (per_w > 1) orth_backtr<4, 2, true>(t.V, A, tau, m, r, s_zb, t.dbg);
        else orth_backtr<4, 1, true>(t.V, A, tau, m, r, s_zb, t.dbg);
      } else {
        if (per_w > 4) orth_backtr<2, 8, false>(t.V, A, tau, m, r, s_zb, t.dbg);
        else if (per_w > 2) orth_backtr<2, 4, false>(t.V, A, tau, m, r, s_zb, t.dbg);
        else if (per_w > 1) orth_backtr<2, 2, false>(t.V, A, tau, m, r, s_zb, t.dbg);
        else orth_backtr<2, 1, false>(t.V, A, tau, m, r, s_zb, t.dbg);
      }
      __syncthreads();
      if (t.dbg && tid == 0) t.dbg[3] = t.dbg[4] = clock64();
      return;
    }
  }
  // modified Gram-Schmidt over the r vectors (warps over later vectors)
  for (int k = 0; k < r; ++k) {
    double *zk = t.V + (int64_t)k * m;
    if (warp == 0) {
      double s2 = 0;
      for (int i = lane; i < m; i += 32) s2 = fma(zk[i], zk[i], s2);
      s2 = frcp(sqrt(warp_sum(s2)));
      for (int i = lane; i < m; i += 32) zk[i] *= s2;
    }
    __syncthreads();
    for (int j = k + 1 + warp; j < r; j += nw) {
      double *zj = t.V + (int64_t)j * m;
      double s2 = 0;
      for (int i = lane; i < m; i += 32) s2 = fma(zk[i], zj[i], s2);
      s2 = warp_sum(s2);
      for (int i = lane; i < m; i += 32) zj[i] -= s2 * zk[i];
    }
    __syncthreads();
  }
  if (t.dbg && tid == 0) t.dbg[3] = clock64();
  // ---- 5. back-transformation V = H_0 ... H_{m-3} Z ----
  if (m <= 256) {
    const int per_w = (r + nw - 1) / nw;
    if (per_w >= 2) backtr_warp<8, 2>(t.V, A, tau, m, r, PRE);
    else backtr_warp<8, 1>(t.V, A, tau, m, r, PRE);
  } else {
    for (int k = warp; k < r; k += nw) {
      double *z = t.V + (int64_t)k * m;
      for (int j = m - 3; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const double *v = A + (PRE ? refl_off(j, m) : (int64_t)j * m);
        double s2 = 0;
        for (int i = j + 1 + lane; i < m; i += 32) s2 = fma(v[i], z[i], s2);
        s2 = warp_sum(s2) * tj;
        for (int i = j + 1 + lane; i < m; i += 32) z[i] -= s2 * v[i];
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (t.dbg && tid == 0) t.dbg[4] = clock64();
}

// ---------------------------------------- PRE pipeline (128 < m <= 512) ----
// Stage 0: eigenvalues of the tridiagonal record over nch CTAs per node.  Every
// CTA scales T, finds lambda_0 (one warp, 32-point multisection) and the
// candidate count (Sturm count at the candidate bound) -- the same arithmetic
// on the same data, so bitwise the same in every CTA -- then multisects its
// slice of the candidates [1, ncomp) with EG lanes per eigenvalue (the more
// CTAs, the more lanes per eigenvalue and the fewer rounds).  Writes lam[k]
// (unscaled) to the record; CTA 0 also lam[0], ||T|| bound, ncomp and the trace.
// The rank (Eq. cutOff1 / curOff6) is decided by k_invit_multi from these.
constexpr int REC_NCOMP = 2, REC_TRACE = 3;   // record slots rec[3 m + .]
__global__ void __launch_bounds__(512, 1) k_eigvals_cl(const EigTask *__restrict__ tasks, double eps, int nch,
                                                       int egmax) {
  extern __shared__ double sh[];
  __shared__ double s_red[32], s_bc[8];
  __shared__ int s_int[4];
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x / nch];
  pdl_wait();
  const int c = blockIdx.x % nch;
  const int m = t.m, mp = (m + 8) & ~7;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *rec = t.work + 6 * (int64_t)m * m;
  if (!(rec[3 * m] > 0.0)) return;   // G = 0: k_invit_multi writes r = 0 (Z4)
  double *d = sh, *e = sh + mp, *e2 = sh + 2 * mp;
  for (int i = tid; i < m; i += blockDim.x) {
    d[i] = rec[i];
    e[i] = rec[m + i];
  }
  __syncthreads();
  double trace = 0.0, fbud = 0.0;
  if (t.frob) {
    double tr = 0.0;
    for (int i = tid; i < m; i += blockDim.x) tr += d[i];
    tr = warp_sum(tr);
    if (lane == 0) s_red[warp] = tr;
    __syncthreads();
    for (int w = 0; w < nw; ++w) trace += s_red[w];
    fbud = eps * eps * (*t.frob) / t.frob_w;
    __syncthreads();
  }
  double gl = 1e300, gu = -1e300, emax2 = 0;
  for (int i = tid; i < m; i += blockDim.x) {
    const double off = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < m - 1 ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - off);
    gu = fmax(gu, d[i] + off);
    if (i < m - 1) {
      e2[i] = e[i] * e[i];
      emax2 = fmax(emax2, e2[i]);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
  }
  if (lane == 0) {
    s_red[warp] = gl;
    s_red[16 + warp] = gu;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 1e300, b = -1e300;
    for (int w = 0; w < nw; ++w) {
      a = fmin(a, s_red[w]);
      b = fmax(b, s_red[16 + w]);
    }
    s_bc[0] = a;
    s_bc[1] = b;
  }
  __syncthreads();
  if (lane == 0) s_red[warp] = emax2;
  __syncthreads();
  double em = 0;
  for (int w = 0; w < nw; ++w) em = fmax(em, s_red[w]);
  gl = s_bc[0];
  gu = s_bc[1];
  const double bnorm = fmax(fabs(gl), fabs(gu));
  const double isc = 1.0 / bnorm;
  __syncthreads();
  for (int i = tid; i < mp; i += blockDim.x) {
    if (i < m) {
      d[i] *= isc;
      if (i < m - 1) e2[i] *= isc * isc;
      else e2[i] = 0.0;
    } else {
      d[i] = 4.0;   // padding: no sign change for x < 4
      e2[i] = 0.0;
    }
  }
  gl *= isc;
  gu *= isc;
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, em * isc * isc) * 1e10;
  gl -= 2.2e-16 * 2 * m + 2 * pivmin;
  gu += 2.2e-16 * 2 * m + 2 * pivmin;
  __syncthreads();
  if (warp == 0) {
    const double l0 = warp_eig_asc(d, e2, m, m - 1, gl, gu, pivmin);
    if (lane == 0) {
      double thr = eps * sqrt(fmax(l0, 0.0));
      thr = 0.25 * thr * thr;
      if (t.frob) thr = fbud / m * isc;   // (scaled) candidate bound of the Frobenius rule
      const int below = sturm_count(d, e2, m, thr, pivmin);
      s_int[0] = min(m, m - below + 1);   // candidates to compute (superset of kept + 1)
      s_bc[2] = l0;
    }
  }
  __syncthreads();
  const int ncomp = s_int[0];
  double *lam = rec + rec_lam_off(m);
  if (c == 0 && tid == 0) {
    lam[0] = s_bc[2] * bnorm;
    rec[3 * m + 1] = bnorm;
    rec[3 * m + REC_NCOMP] = (double)ncomp;
    rec[3 * m + REC_TRACE] = trace;
  }
  const int per = (ncomp - 1 + nch - 1) / nch, k1 = 1 + c * per, k2 = min(ncomp, k1 + per);
  if (k1 >= k2) return;
  // lanes per eigenvalue: many (few rounds) for the latency-bound cluster path;
  // egmax = 2 for the throughput path (many nodes per SM: the fewest Sturm
  // steps per eigenvalue)
  const int cnt = k2 - k1, lanes = (int)blockDim.x;
  int eg = cnt * 32 <= lanes ? 32 : (cnt * 16 <= lanes ? 16 : (cnt * 8 <= lanes ? 8 : 4));
  if (eg > egmax) eg = egmax;
  if (eg < 2 && egmax >= 2) eg = 2;
  switch (eg) {
    case 32: grp_multisect<32>(d, e2, m, k1, k2, gl, gu, pivmin, lam, bnorm); break;
    case 16: grp_multisect<16>(d, e2, m, k1, k2, gl, gu, pivmin, lam, bnorm); break;
    case 8: grp_multisect<8>(d, e2, m, k1, k2, gl, gu, pivmin, lam, bnorm); break;
    case 4: grp_multisect<4>(d, e2, m, k1, k2, gl, gu, pivmin, lam, bnorm); break;
    case 2: grp_multisect<2>(d, e2, m, k1, k2, gl, gu, pivmin, lam, bnorm); break;
    default: grp_multisect<1>(d, e2, m, k1, k2, gl, gu, pivmin, lam, bnorm); break;
  }
}

// Stage 1: the rank from the eigenvalues (Eq. cutOff1, or Eq. curOff6 with the
// trace), then inverse iteration for the kept eigenvalues of the tridiagonal
// record, one CTA per chunk of vectors (chunk c: k in [c nb, (c+1) nb) ∩ [0, r)),
// each chunk's LU / right-hand sides in shared memory; grid = nodes x nch.
// CTA 0 of each node writes sigma and the rank.
__global__ void __launch_bounds__(256) k_invit_multi(const EigTask *__restrict__ tasks, int nch, int smem_cap_doubles,
                                                     double eps) {
  pdl_trigger();
  extern __shared__ double sh[];
  const EigTask t = tasks[blockIdx.x / nch];
  pdl_wait();   // task descriptors are static: read before the wait
  const int c = blockIdx.x % nch;
  const int m = t.m;
  const double *rec = t.work + 6 * (int64_t)m * m;
  int r = 0, ncomp = 0;
  {
    __shared__ int s_cnt;
    const double *lg = rec + rec_lam_off(m);
    const bool live = rec[3 * m] > 0.0;
    ncomp = live ? (int)rec[3 * m + REC_NCOMP] : 0;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    if (t.frob) {   // smallest k with tail(k) = trace - sum_{t<k} lambda_t < budget
      if (threadIdx.x == 0 && live) {
        const double trace = rec[3 * m + REC_TRACE], fbud = eps * eps * (*t.frob) / t.frob_w;
        double pre = 0.0;
        int k = 0;
        while (k < ncomp && !(trace - pre < fbud)) pre += fmax(lg[k++], 0.0);
        s_cnt = k;
      }
    } else if (live) {
      const double sig0 = sqrt(fmax(lg[0], 0.0));
      int cn = 0;
      for (int k = threadIdx.x; k < ncomp; k += blockDim.x) cn += (sqrt(fmax(lg[k], 0.0)) >= eps * sig0);
      if (cn) atomicAdd(&s_cnt, cn);
    }
    __syncthreads();
    r = s_cnt;
    if (c == 0) {
      for (int k = threadIdx.x; k < m; k += blockDim.x) t.sig[k] = (k < ncomp) ? sqrt(fmax(lg[k], 0.0)) : 0.0;
      if (threadIdx.x == 0) *t.rank_out = r;
    }
  }
  const int64_t per = 5 * (int64_t)m + (m + 7) / 8;
  const int mp = (m + 8) & ~7;
  const int nb = (int)min((int64_t)blockDim.x, ((int64_t)smem_cap_doubles - 2 * mp) / per);
  const int k0 = c * nb;
  if (k0 >= r || nb <= 0) return;
  const int nbc = min(nb, r - k0);
  double *d = sh, *e = sh + mp, *ws = sh + 2 * mp;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    d[i] = rec[i];
    e[i] = rec[m + i];
  }
  __syncthreads();
  const double *lam = rec + rec_lam_off(m);
  const double pertol = 10.0 * 2.2e-16 * rec[3 * m + 1];
  const int kk = threadIdx.x;
  if (kk < nbc) {
    const int k = k0 + kk;
    double sft = lam[k];
    for (int q = 1; q <= k && lam[k - q] - lam[k] < pertol; ++q) sft -= pertol;
    double *DL = ws + kk, *Dv = DL + (int64_t)m * nbc, *DU = Dv + (int64_t)m * nbc, *DU2 = DU + (int64_t)m * nbc,
           *bb = DU2 + (int64_t)m * nbc;
    unsigned char *pv = reinterpret_cast<unsigned char *>(ws + 5 * (int64_t)m * nbc) + kk;
    invit_one(d, e, m, sft, pertol, k, DL, Dv, DU, DU2, bb, pv, nbc, t.V + (int64_t)k * m);
  }
}

// Throughput path (waves of many nodes with m <= 128, after k_tridiag_reg,
// k_eigvals_cl and k_invit_multi): MGS + back-transformation of one node per
// 256-thread CTA, vectors in registers, the packed reflectors of the record
// staged through shared memory; several nodes share an SM.
template <int NV>
__device__ __forceinline__ void orthbt_node(const EigTask &t, int m, int r, double *sh, int stg_cap) {
  const double *rec = t.work + 6 * (int64_t)m * m;
  double *tau = sh, *zb = sh + 136, *stg = zb + 256;
  for (int i = threadIdx.x; i < m; i += blockDim.x) tau[i] = rec[2 * m + i];
  __syncthreads();
  orth_backtr<4, NV, true>(t.V, rec + 4 * (int64_t)m, tau, m, r, zb, nullptr, stg, stg_cap);
}
constexpr int ORTHBT_STG = 4096;   // reflector staging doubles per CTA
constexpr size_t ORTHBT_SMEM = (size_t)(136 + 256 + ORTHBT_STG) * 8;
__global__ void __launch_bounds__(256, 2) k_orthbt(const EigTask *__restrict__ tasks) {
  extern __shared__ double sh[];
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x];
  pdl_wait();
  const int m = t.m, r = *t.rank_out;
  if (r <= 0 || m > 128) return;
  const int per_w = (r + 7) / 8;
  if (per_w <= 1) orthbt_node<1>(t, m, r, sh, ORTHBT_STG);
  else if (per_w <= 2) orthbt_node<2>(t, m, r, sh, ORTHBT_STG);
  else if (per_w <= 4) orthbt_node<4>(t, m, r, sh, ORTHBT_STG);
  else if (per_w <= 8) orthbt_node<8>(t, m, r, sh, ORTHBT_STG);
  else orthbt_node<16>(t, m, r, sh, ORTHBT_STG);
}

// Block Gram-Schmidt of the r inverse-iteration vectors over a cluster of CL
// CTAs (round 1: MGS with one cluster barrier per vector): CTA c
// owns the panel of vectors [c rb, (c+1) rb) (rb = ceil(r / CL) <= 32), two
// per warp, in registers (lane's rows 32 q + lane).  For c = 0 .. CL-1:
//   CTA c orthonormalises its panel by MGS inside the CTA (pivot vector l in
//   warp l mod 16, broadcast through shared memory: one block barrier per
//   vector), writing the final vectors to V; one cluster barrier; every later
//   CTA stages panel c from L2 and removes it from its own vectors (block
//   classical Gram-Schmidt, 8 columns per warp reduction).
// Selective reorthogonalisation (Kahan-Parlett): a pivot whose norm fell below
// 1/sqrt(2) of its norm as produced by inverse iteration is projected once more
// against every earlier final vector (all 16 warps, partial corrections
// summed in shared memory) before it is normalised; so clusters of close
// eigenvalues, whose inverse-iteration vectors are nearly parallel, still come
// out orthonormal to working precision (single-pass MGS lost up to 1e-7 there).
// Dynamic shared memory: 32 (m|1) staging + 2 x 512 pivot + 512 + 16 x 512
// partial corrections (doubles) at the QM class's maximum m.
template <int QM>
constexpr int orth_bgs_smem_doubles() {
  return 32 * (32 * QM + 1) + 2 * 32 * QM + 32 * QM + 16 * 32 * QM;
}
template <int QM, int CL>
__global__ void __launch_bounds__(512, 1) k_orth_bgs(const EigTask *__restrict__ tasks) {
  extern __shared__ double sh[];
  __shared__ int s_flag[2];
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int MX = 32 * QM;
  const int rank = (int)cl.block_rank();
  const EigTask t = tasks[blockIdx.x / CL];
  const int m = t.m, r = *t.rank_out;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (r <= 0) return;   // uniform over the cluster
  const int rb = (r + CL - 1) / CL, j0 = rank * rb, nown = max(0, min(r, j0 + rb) - j0);
  const int ldz = m | 1;
  double *stage = sh, *pbuf = sh + 32 * (MX + 1), *zks = pbuf + 2 * MX, *red = zks + MX;
  double *V = t.V;
  double z[2][QM], n0[2];
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const int l = warp + 16 * v;
    double a = 0.0;
#pragma unroll
    for (int q = 0; q < QM; ++q) {
      const int i = 32 * q + lane;
      z[v][q] = (l < nown && i < m) ? V[(int64_t)(j0 + l) * m + i] : 0.0;
      a = fma(z[v][q], z[v][q], a);
    }
    n0[v] = warp_sum(a);
  }
  const bool prof = t.dbg && rank == 1 && threadIdx.x == 0;
  long long pa[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pc = prof ? clock64() : 0;
#define OBGS_PROF(i) if (prof) { const long long tn = clock64(); pa[i] += tn - pc; pc = tn; }
  for (int c = 0; c < CL && c * rb < r; ++c) {
    if (rank == c) {
      // n2: the pivot's squared norm, carried from the previous step's update
      // (||z - s q||^2 = z.z - s^2 from the same warp reduction as s; exact
      // to ~2u relative while no reorthogonalisation is due, i.e. while
      // ||z'||^2 >= ||z_0||^2 / 2), so each vector costs one block barrier
      double n2 = 0.0;
      if (nown > 0 && warp == 0) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < QM; ++q) a = fma(z[0][q], z[0][q], a);
        n2 = warp_sum(a);
      }
      for (int l = 0; l < nown; ++l) {
        const int pw = l & 15, k = j0 + l;
        const bool sel = (l >> 4) != 0;
        double *pb = pbuf + (l & 1) * MX;
        auto finish = [&]() {   // pivot warp: normalise, publish to the CTA and to V
          const double inv = n2 > 0.0 ? frsqrt(n2) : 0.0;
#pragma unroll
          for (int q = 0; q < QM; ++q) {
            const int row = 32 * q + lane;
            double x;
            if (sel) x = (z[1][q] *= inv);
            else x = (z[0][q] *= inv);
            pb[row] = x;
            if (row < m) V[(int64_t)k * m + row] = x;
          }
        };
        if (warp == pw) {
          const bool need = n2 < 0.5 * (sel ? n0[1] : n0[0]) && k > 0;
          if (need) {
#pragma unroll
            for (int q = 0; q < QM; ++q) zks[32 * q + lane] = sel ? z[1][q] : z[0][q];
          } else {
            finish();
          }
          if (lane == 0) s_flag[l & 1] = need;
        }
        OBGS_PROF(4)
        __syncthreads();
        if (s_flag[l & 1]) {   // uniform: reproject the pivot on every earlier final vector
          double *corr = red + warp * MX + lane;   // this warp's partial correction
#pragma unroll
          for (int q = 0; q < QM; ++q) corr[32 * q] = 0.0;
          for (int i = warp; i < k; i += 16) {
            double qv[QM], d = 0.0;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
              const int row = 32 * q + lane;
              qv[q] = row < m ? __ldcg(V + (int64_t)i * m + row) : 0.0;
              d = fma(qv[q], zks[row], d);
            }
            d = warp_sum(d);
#pragma unroll
            for (int q = 0; q < QM; ++q) corr[32 * q] = fma(d, qv[q], corr[32 * q]);
          }
          __syncthreads();
          if (warp == pw) {
            double a = 0.0;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
              double sacc = 0.0;
              for (int w = 0; w < 16; ++w) sacc += red[w * MX + 32 * q + lane];
              if (sel) {
                z[1][q] -= sacc;
                a = fma(z[1][q], z[1][q], a);
              } else {
                z[0][q] -= sacc;
                a = fma(z[0][q], z[0][q], a);
              }
            }
            n2 = warp_sum(a);
            finish();
          }
          __syncthreads();
        }
        OBGS_PROF(5)
        // remove the pivot from this CTA's later vectors (only warps holding
        // one: shuffles are a shared, low-throughput resource); the warp of the
        // next pivot also forms that vector's new squared norm
        const int ln = l + 1;
        const bool nxt = ln < nown && warp == (ln & 15), nsel = (ln >> 4) != 0;
        const bool u0 = warp > l && warp < nown, u1 = warp + 16 > l && warp + 16 < nown;
        if (u0 || u1) {
          double pq[QM], s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int q = 0; q < QM; ++q) {
            pq[q] = pb[32 * q + lane];
            s4[0] = fma(pq[q], z[0][q], s4[0]);
            s4[1] = fma(pq[q], z[1][q], s4[1]);
          }
          if (nxt) {
            double a = 0.0;
#pragma unroll
            for (int q = 0; q < QM; ++q) a = fma(nsel ? z[1][q] : z[0][q], nsel ? z[1][q] : z[0][q], a);
            s4[2] = a;
          }
          if (u1) {
            warp_sum_multi<4>(s4);
          } else if (nxt) {
            double s2[2] = {s4[0], s4[2]};
            warp_sum_multi<2>(s2);
            s4[0] = s2[0];
            s4[2] = s2[1];
          } else {
            s4[0] = warp_sum(s4[0]);
          }
#pragma unroll
          for (int q = 0; q < QM; ++q) {
            if (u0) z[0][q] = fma(-s4[0], pq[q], z[0][q]);
            if (u1) z[1][q] = fma(-s4[1], pq[q], z[1][q]);
          }
          if (nxt) {
            const double sn = nsel ? s4[1] : s4[0];
            n2 = fma(-sn, sn, s4[2]);
          }
        }
        OBGS_PROF(6)
      }
    }
    OBGS_PROF(0)
    cl.sync();   // panel c final in V, visible to the cluster
    OBGS_PROF(1)
    if (rank > c) {
      const int c0 = c * rb, nc = min(r, c0 + rb) - c0;
      for (int e = threadIdx.x; e < nc * m; e += blockDim.x) {
        const int i = e / m, row = e - i * m;
        stage[i * ldz + row] = __ldcg(V + (int64_t)(c0 + i) * m + row);
      }
      __syncthreads();
      OBGS_PROF(2)
      const bool has0 = warp < nown, has1 = warp + 16 < nown;
      if (has0 && !has1) {   // one vector in this warp: 8 columns per reduction
        for (int i0 = 0; i0 < nc; i0 += 8) {
          double s8[8];
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) {
            const int i = i0 + ii;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
              const int row = 32 * q + lane;
              const double qv = (i < nc && row < m) ? stage[i * ldz + row] : 0.0;
              if (q & 1) a1 = fma(qv, z[0][q], a1);
              else a0 = fma(qv, z[0][q], a0);
            }
            s8[ii] = a0 + a1;
          }
          warp_sum_multi<8>(s8);
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) {
            const int i = i0 + ii;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
              const int row = 32 * q + lane;
              const double qv = (i < nc && row < m) ? stage[i * ldz + row] : 0.0;
              z[0][q] = fma(-s8[ii], qv, z[0][q]);
            }
          }
        }
      } else if (has1)
      for (int i0 = 0; i0 < nc; i0 += 8) {
        double s16[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) s16[u] = 0.0;
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
          const int i = i0 + ii;
#pragma unroll
          for (int q = 0; q < QM; ++q) {
            const int row = 32 * q + lane;
            const double qv = (i < nc && row < m) ? stage[i * ldz + row] : 0.0;
            s16[ii] = fma(qv, z[0][q], s16[ii]);
            s16[8 + ii] = fma(qv, z[1][q], s16[8 + ii]);
          }
        }
        warp_sum_multi<16>(s16);
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
          const int i = i0 + ii;
#pragma unroll
          for (int q = 0; q < QM; ++q) {
            const int row = 32 * q + lane;
            const double qv = (i < nc && row < m) ? stage[i * ldz + row] : 0.0;
            z[0][q] = fma(-s16[ii], qv, z[0][q]);
            z[1][q] = fma(-s16[8 + ii], qv, z[1][q]);
          }
        }
      }
      __syncthreads();   // the staging buffer is refilled next round
      OBGS_PROF(3)
    }
  }
  if (prof)
    for (int q = 0; q < 8; ++q) t.dbg[20 + q] = pa[q];
#undef OBGS_PROF
}

// Back-transformation V = H_0 ... H_{m-3} Z for a chunk of 16 NV vectors per
// CTA (register-resident, reflectors staged through shared memory in
// contiguous packed segments); grid = nodes x nch.
template <int Q, int NV>
__global__ void __launch_bounds__(512) k_backtr_multi(const EigTask *__restrict__ tasks, int nch, int smem_cap_doubles) {
  pdl_trigger();
  extern __shared__ double sh[];
  const EigTask t = tasks[blockIdx.x / nch];
  pdl_wait();   // task descriptors are static: read before the wait
  const int c = blockIdx.x % nch;
  const int m = t.m, r = *t.rank_out;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int k0 = c * nw * NV;
  if (k0 >= r) return;
  const double *rec = t.work + 6 * (int64_t)m * m;
  double *tau = sh;
  double *stg = sh + ((m + 8) & ~7);
  const int stg_cap = smem_cap_doubles - ((m + 8) & ~7);
  for (int i = threadIdx.x; i < m; i += blockDim.x) tau[i] = rec[2 * m + i];
  const double *A = rec + 4 * (int64_t)m;
  double z[NV][Q];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int k = k0 + warp + v * nw;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      z[v][q] = (k < r && i < m) ? t.V[(int64_t)k * m + i] : 0.0;
    }
  }
  const int ch = max(1, stg_cap / max(m, 1));
  for (int jc = m - 3; jc >= 0; jc -= ch) {
    const int jl = max(0, jc - ch + 1);
    const int64_t lo = refl_off(jl, m) + jl + 1, hi = refl_off(jc, m) + m;
    __syncthreads();
    for (int64_t q = lo + threadIdx.x; q < hi; q += blockDim.x) stg[q - lo] = A[q];
    __syncthreads();
    const double *base = stg - lo;
    for (int j = jc; j >= jl; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double *vj = base + refl_off(j, m);
      double vv[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int i = lane + 32 * q;
        vv[q] = (i > j && i < m) ? vj[i] : 0.0;
      }
      double s[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        s[v] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) s[v] = fma(vv[q], z[v][q], s[v]);
      }
      warp_sum_multi<NV>(s);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double sv = s[v] * tj;
#pragma unroll
        for (int q = 0; q < Q; ++q) z[v][q] = fma(-sv, vv[q], z[v][q]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int k = k0 + warp + v * nw;
    if (k < r)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int i = lane + 32 * q;
        if (i < m) t.V[(int64_t)k * m + i] = z[v][q];
      }
  }
}

// ---- f1: rank-revealing QR compressor (P:l.616, P:l.840) ----
// Column-pivoted (Businger-Golub) QR of the stack M, M P = Q R, computed as
// the diagonal-pivoted Cholesky of the Gram G = M^T M = P R^T R P^T (the pivot
// "largest remaining column norm of M" is "largest remaining diagonal of the
// Schur complement of G").  Truncated at the first k with R_kk < eps R_00
// (reading F1); V = an orthonormal basis of span(R[:r, :] P^T)^T = span(L),
// L = the m x r Cholesky columns in the original index order, by classical
// Gram-Schmidt with reorthogonalisation (CGS2).  One CTA (512 threads) per
// node, thread j owns row j (m <= 512); left-looking: column k of L is
// G[:, p] - L[:, :k] L[p, :k]^T, read from the L2-resident output V.
// Writes V (m x r, ld m), sig (R_kk for k < r, the first dropped R_kk at r,
// zeros after), *rank_out.  G = 0 -> r = 0 (Z4); eps = 0 -> V = I, r = m (Z3).
constexpr int RRQR_MAXM = 512;
// NT threads, thread j owns row j (m <= NT).  G and L stay in global memory
// (L2-resident; measured faster than staging them in shared memory, which
// costs occupancy on the many-node waves).
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_rrqr(const EigTask *__restrict__ tasks, double eps, int *status) {
  __shared__ double s_v[NT / 32];
  __shared__ int s_i[NT / 32];
  __shared__ double Lp[RRQR_MAXM];     // row p of L (pivoted row) / CGS coefficients
  __shared__ double s_bc[2];
  __shared__ int s_p;
  pdl_trigger();
  const EigTask t = tasks[blockIdx.x];
  pdl_wait();
  const int m = t.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = NT / 32;
  const int j = tid;
  const bool row = j < m;
  const double *G = t.G;
  double *Vw = t.V;                    // L, then V (column-major, ld m)
  double dj = row ? G[j + (int64_t)j * m] : 0.0;   // remaining diagonal
  bool done = !row;
  // block argmax of the remaining diagonal (ties -> smallest index)
  auto argmax = [&](double v, int idx) {
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (v2 > v || (v2 == v && i2 < idx)) {
        v = v2;
        idx = i2;
      }
    }
    if (lane == 0) {
      s_v[warp] = v;
      s_i[warp] = idx;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = s_v[0];
      int bi = s_i[0];
      for (int w = 1; w < nw; ++w)
        if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < bi)) {
          bv = s_v[w];
          bi = s_i[w];
        }
      s_bc[0] = bv;
      s_p = bi;
    }
    __syncthreads();
  };
  if (eps == 0.0) {
    argmax(row ? dj : -1.0, row ? j : 1 << 30);
    const bool zero = !(s_bc[0] > 0.0);
    for (int64_t q = tid; q < (int64_t)m * m; q += NT) t.V[q] = ((q % m) == (q / m)) ? 1.0 : 0.0;
    for (int q = tid; q < m; q += NT) t.sig[q] = 0.0;
    if (tid == 0) *t.rank_out = zero ? 0 : m;
    return;
  }
  double r00 = 0.0;
  int r = 0;
  for (int k = 0; k < m; ++k) {
    argmax(done ? -1.0 : dj, done ? (1 << 30) : j);
    const double dmax = s_bc[0];
    const int p = s_p;
    const double rkk = sqrt(fmax(dmax, 0.0));
    if (k == 0) r00 = rkk;
    if (!(rkk > 0.0) || rkk < eps * r00) {   // truncation (uniform)
      if (tid == 0) t.sig[k] = rkk;
      break;
    }
    if (tid == 0) t.sig[k] = rkk;
    for (int i = tid; i < k; i += NT) Lp[i] = Vw[p + (int64_t)i * m];
    __syncthreads();
    double l = 0.0;
    if (row && !done) {
      if (j == p) {
        l = rkk;
        done = true;
      } else {
        double s0 = G[j + (int64_t)p * m], s1 = 0.0;
        int i = 0;
        for (; i + 1 < k; i += 2) {
          s0 = fma(-Vw[j + (int64_t)i * m], Lp[i], s0);
          s1 = fma(-Vw[j + (int64_t)(i + 1) * m], Lp[i + 1], s1);
        }
        if (i < k) s0 = fma(-Vw[j + (int64_t)i * m], Lp[i], s0);
        l = (s0 + s1) * frcp(rkk);
        dj -= l * l;
      }
    }
    if (row) Vw[j + (int64_t)k * m] = l;
    r = k + 1;
    __syncthreads();   // column k visible before the next step reads row p of L
  }
  for (int q = r + 1 + tid; q < m; q += NT) t.sig[q] = 0.0;
  if (tid == 0) *t.rank_out = r;
  if (r == 0) return;
  // ---- V = orth(L): CGS2 (two projections per column), column k by the block ----
  for (int k = 0; k < r; ++k) {
    double *vk = Vw + (int64_t)k * m;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = warp; i < k; i += nw) {   // coefficients against the finished columns
        const double *vi = Vw + (int64_t)i * m;
        double sacc = 0.0;
        for (int q = lane; q < m; q += 32) sacc = fma(vi[q], vk[q], sacc);
        sacc = warp_sum(sacc);
        if (lane == 0) Lp[i] = sacc;
      }
      __syncthreads();
      if (row && k > 0) {
        double s0 = 0.0, s1 = 0.0;
        int i = 0;
        for (; i + 1 < k; i += 2) {
          s0 = fma(Vw[j + (int64_t)i * m], Lp[i], s0);
          s1 = fma(Vw[j + (int64_t)(i + 1) * m], Lp[i + 1], s1);
        }
        if (i < k) s0 = fma(Vw[j + (int64_t)i * m], Lp[i], s0);
        vk[j] -= s0 + s1;
      }
      __syncthreads();
    }
    // normalise
    double ss = row ? vk[j] * vk[j] : 0.0;
    ss = warp_sum(ss);
    if (lane == 0) s_v[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double a = 0.0;
      for (int w = 0; w < nw; ++w) a += s_v[w];
      s_bc[1] = a > 0.0 ? 1.0 / sqrt(a) : 0.0;
    }
    __syncthreads();
    if (row) vk[j] *= s_bc[1];
    __syncthreads();
  }
  (void)status;
}

// ----------------------------------------------------------------- pivot ----
// (k_eig_t<true> for m <= 128, k_eig_t<false> otherwise)

// Fused pivot of (s, b): K = [[S, V], [V^T, 0]] (n = m + r) factored as
// K = L D L^T with D = diag(I_m, -I_r) (Cholesky of S, then of
// W = V^T S^{-1} V for the black node, P:l.396-399), then overwritten by
// L^{-1} (lower, strict upper zeroed).  Works in shared memory when n^2 fits.
struct PivTask {
  double *F;  // n x n at ld
  int ld, m, r, node;
  double *F2;  // LU path: where U^{-T} goes (nullptr: F + ld * n, the record's region 1)
  int pivot;   // LU path (k_pivot_lu): partial pivoting (see there); 0 = none
  // k_pivot_blk as the diagonal-block step of the blocked large pivot: when Xo
  // is set, L^{-1} goes to Xo (ld ldxo, upper triangle zeroed) and
  // Wt = L^{-T} D (64 x 64, ld 64) instead of back into F
  double *Xo, *Wt;
  int ldxo;
};

// LU path without pivoting: a multiplier |l_ij| above this (partial pivoting
// keeps |l_ij| <= 1), or a vanishing pivot, reports LORASP_NEED_PIVOT; the host
// then re-runs the sweep with partial pivoting (k_pivot_lu, pivot = 1).
constexpr double LU_GROWTH_MAX = 64.0;
constexpr int LORASP_NEED_PIVOT = -10;   // internal status, never returned by the C ABI

// block-wide max of v (all threads get it); red: >= 16 doubles of shared scratch
__device__ __forceinline__ double block_max(double v, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = 0;
  for (int w = 0; w < nw; ++w) v = fmax(v, red[w]);
  return v;
}
// growth of the multipliers max |l_ij| (strict lower of A, n x n at lda); every
// thread returns it; the largest seen is kept in status[2..3] (a double)
__device__ __forceinline__ double lu_growth(const double *A, int lda, int n, double *red, int *status) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double g = 0;
  for (int j = warp; j < n; j += nw)
    for (int i = j + 1 + lane; i < n; i += 32) g = fmax(g, fabs(A[i + (int64_t)j * lda]));
  g = block_max(g, red);
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long *>(status + 2), (unsigned long long)__double_as_longlong(g));
  return g;
}

__global__ void __launch_bounds__(512) k_pivot(const PivTask *__restrict__ tasks,
                                               int smem_cap_doubles, int *status) {
  pdl_trigger();
  extern __shared__ double sh[];
  const PivTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
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
    for (int j = warp; j < n; j += nw)
      for (int i = lane; i < n; i += 32) A[i + (int64_t)j * n] = (i >= j) ? t.F[i + (int64_t)j * t.ld] : 0.0;
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
    const double sc = d * frcp(lkk);
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
    const double ajj = frcp(A[j + (int64_t)j * lda]);
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
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i < n; i += 32) {
      double v = (i >= j) ? A[i + (int64_t)j * lda] : 0.0;
      t.F[i + (int64_t)j * t.ld] = v;
    }
}

// --------------------------------------------------------- LU pivot (general) ----
// LU path: the fused pivot K = [[S, V], [V^T, 0]] (n = m + r, full, ld) is
// factored P K = L U, then region 0 <- L^{-1} P and region 1 <- U^{-T} (lower),
// so that K^{-1} = U^{-1} (L^{-1} P): the Z GEMM X = (L^{-1} P) C and the apply's
// forward step y = (L^{-1} P)[:, :m] rhs use region 0 as a general matrix.
// pivot = 0: no pivoting (P = I; region 0 unit lower); a vanishing pivot or a
//   multiplier above LU_GROWTH_MAX reports LORASP_NEED_PIVOT.
// pivot = 1: partial pivoting restricted to the two diagonal blocks -- rows of
//   [0, m) for the columns of S, rows of [m, n) for the Schur block -- i.e.
//   P = diag(P1, P2): exactly the oracle's Eliminate(s) then Eliminate(b), each
//   with a partial-pivot LU (P:l.101-106, P:l.396-399; reading Z11).  A vanishing
//   pivot then is LORASP_E_SINGULAR_PIVOT.
// Shared memory when n^2 + 2n fits (A, tmp, the permutation), else in place in
// region 0 (global), with per-warp row strips for the final column permutation.
__global__ void __launch_bounds__(512) k_pivot_lu(const PivTask *__restrict__ tasks, int smem_cap_doubles,
                                                  int *status) {
  pdl_trigger();
  extern __shared__ double sh[];
  const PivTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ int s_fail, s_p;
  __shared__ double s_red[16];
  const bool in_smem = (int64_t)n * n + 2 * (int64_t)n <= smem_cap_doubles;
  double *tmp = sh;
  int *perm = reinterpret_cast<int *>(sh + n);   // n ints
  double *A;
  int lda;
  if (in_smem) {
    A = sh + 2 * n;
    lda = n;
    for (int j = warp; j < n; j += nw)
      for (int i = lane; i < n; i += 32) A[i + (int64_t)j * n] = t.F[i + (int64_t)j * t.ld];
  } else {
    A = t.F;
    lda = t.ld;
  }
  for (int i = tid; i < n; i += blockDim.x) perm[i] = i;
  if (tid == 0) s_fail = 0;
  __syncthreads();
  double amax = 0;   // scale for the singularity test
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i < n; i += 32) amax = fmax(amax, fabs(A[i + (int64_t)j * lda]));
  amax = block_max(amax, s_red);
  const int fail_code = t.pivot ? -3 : LORASP_NEED_PIVOT;
  // right-looking LU
  for (int k = 0; k < n; ++k) {
    if (t.pivot) {
      const int e = (k < t.m) ? t.m : n;   // candidate rows [k, e)
      if (warp == 0) {
        double best = -1.0;
        int bi = k;
        for (int i = k + lane; i < e; i += 32) {
          const double v = fabs(A[i + (int64_t)k * lda]);
          if (v > best) {
            best = v;
            bi = i;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {   // max |a|, ties -> smaller row
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        if (lane == 0) {
          s_p = bi;
          if (bi != k) {
            const int q = perm[k];
            perm[k] = perm[bi];
            perm[bi] = q;
          }
        }
      }
      __syncthreads();
      const int p = s_p;
      if (p != k)
        for (int j = tid; j < n; j += blockDim.x) {   // whole rows (L part included)
          const double a = A[k + (int64_t)j * lda];
          A[k + (int64_t)j * lda] = A[p + (int64_t)j * lda];
          A[p + (int64_t)j * lda] = a;
        }
      __syncthreads();
    }
    const double piv = A[k + (int64_t)k * lda];
    if (!(fabs(piv) > 1e-14 * amax) || !isfinite(piv)) {
      if (tid == 0) {
        s_fail = 1;
        if (atomicCAS(&status[0], 0, fail_code) == 0) status[1] = t.node;
      }
      break;
    }
    const double rp = frcp(piv);
    __syncthreads();
    for (int i = k + 1 + tid; i < n; i += blockDim.x) A[i + (int64_t)k * lda] *= rp;
    __syncthreads();
    for (int j = k + 1 + warp; j < n; j += nw) {
      const double ukj = A[k + (int64_t)j * lda];
      double *cj = A + (int64_t)j * lda;
      const double *ck = A + (int64_t)k * lda;
      for (int i = k + 1 + lane; i < n; i += 32) cj[i] = fma(-ck[i], ukj, cj[i]);
    }
    __syncthreads();
  }
  if (s_fail) return;
  if (!t.pivot && lu_growth(A, lda, n, s_red, status) > LU_GROWTH_MAX) {
    if (tid == 0 && atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
    return;
  }
  // U^{-1} in place (upper incl. diagonal), columns ascending:
  // u_jj <- 1/u_jj; A[0:j, j] <- -u_jj^{-1} * Uinv[0:j, 0:j] A[0:j, j]
  for (int j = 0; j < n; ++j) {
    for (int i = tid; i < j; i += blockDim.x) tmp[i] = A[i + (int64_t)j * lda];
    __syncthreads();
    const double ajj = frcp(A[j + (int64_t)j * lda]);
    for (int i = tid; i < j; i += blockDim.x) {
      double sacc = 0;
      for (int k = i; k < j; ++k) sacc = fma(A[i + (int64_t)k * lda], tmp[k], sacc);
      A[i + (int64_t)j * lda] = -ajj * sacc;
    }
    __syncthreads();
    if (tid == 0) A[j + (int64_t)j * lda] = ajj;
    __syncthreads();
  }
  // region 1 <- U^{-T} (lower): (U^{-T})(i, j) = U^{-1}(j, i) for i >= j
  double *R1 = t.F2 ? t.F2 : t.F + (int64_t)t.ld * n;
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i < n; i += 32) R1[i + (int64_t)j * t.ld] = (i >= j) ? A[j + (int64_t)i * lda] : 0.0;
  __syncthreads();
  // L^{-1} in place (strict lower, unit diagonal), columns descending
  for (int j = n - 1; j >= 0; --j) {
    for (int i = j + 1 + tid; i < n; i += blockDim.x) tmp[i] = A[i + (int64_t)j * lda];
    __syncthreads();
    for (int i = j + 1 + tid; i < n; i += blockDim.x) {
      double sacc = tmp[i];   // unit diagonal of L^{-1} at (i, i)
      for (int k = j + 1; k < i; ++k) sacc = fma(A[i + (int64_t)k * lda], tmp[k], sacc);
      A[i + (int64_t)j * lda] = -sacc;
    }
    __syncthreads();
  }
  // region 0 <- L^{-1} P: column perm[k] of L^{-1} P is column k of L^{-1}
  if (in_smem || !t.pivot) {
    for (int j = warp; j < n; j += nw)
      for (int i = lane; i < n; i += 32) {
        const double v = (i > j) ? A[i + (int64_t)j * lda] : (i == j ? 1.0 : 0.0);
        t.F[i + (int64_t)perm[j] * t.ld] = v;
      }
  } else {   // in place: each warp permutes whole rows through its strip of n doubles
    double *strip = sh + 2 * n + (int64_t)warp * n;
    for (int i = warp; i < n; i += nw) {
      for (int k = lane; k < n; k += 32) strip[k] = (i > k) ? A[i + (int64_t)k * lda] : (i == k ? 1.0 : 0.0);
      __syncwarp();
      for (int k = lane; k < n; k += 32) t.F[i + (int64_t)perm[k] * t.ld] = strip[k];
      __syncwarp();
    }
  }
}

// ----------------------------------------------- blocked pivot (one CTA) ----
// Same result as k_pivot (K = L D L^T, then L^{-1}), for n <= PIVB_MAXN in
// shared memory, with 16-column blocks so that the number of block barriers is
// ~5 per block instead of ~5 per column:
//   factor: warp 0 factors the 16x16 diagonal block and inverts it (warp-
//   synchronous), every thread solves one row of the panel
//   L21 = A21 L11^{-T} D1, warps update the trailing lower triangle
//   A22 -= L21 D1 L21^T;
//   invert (in place, blocks descending): T = X22 L21 (X22 already inverted)
//   is parked transposed in the free upper triangle, A21 <- -T L11^{-1},
//   A11 <- L11^{-1}.
constexpr int PIVB_NB = 16;
constexpr int PIVB_MAXN = 160;

// signed Cholesky of the b x b diagonal block at j0 by one warp with the block
// in registers (lane = row, columns by shuffles): no shared-memory round trip
// per column step.  rd[j0 + k] <- 1 / l_kk.  Returns false on a non-positive
// pivot (uniform across the warp).
__device__ __forceinline__ bool pivb_diag_chol(double *__restrict__ A, int lda, int j0, int b, int m,
                                               double *__restrict__ rd, int lane, double *lcol) {
  // Branch-free (selects only, so no reconvergence points on the chain): column
  // k's multipliers reach the other rows through shared memory (lcol, >= 33
  // doubles; every lane writes its slot) instead of 15 shuffles; a failure is
  // accumulated rather than breaking out of the unrolled loop.
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
      ok = ok && (v > 0.0) && isfinite(v);
      const double rk = frsqrt(fmax(v, 1e-300));
      const double lik = (i > k) ? a[k] * (d * rk) : 0.0;
      a[k] = (i == k) ? v * rk : ((i > k) ? lik : a[k]);
      rd[j0 + k] = rk;   // every lane stores the same value
      lcol[i] = lik;
      __syncwarp();
      const double f = -d * lik;
#pragma unroll
      for (int jj = k + 1; jj < PIVB_NB; ++jj) {
        const double u = fma(f, lcol[jj], a[jj]);
        a[jj] = (jj < b && i >= jj) ? u : a[jj];
      }
      __syncwarp();
    }
  }
  if (ok) {
#pragma unroll
    for (int c = 0; c < PIVB_NB; ++c)
      if (i < b && c <= i) A[(j0 + i) + (j0 + c) * lda] = a[c];
  }
  __syncwarp();
  return ok;
}

__device__ __forceinline__ void pivb_diag_inverse(const double *__restrict__ A, int lda, int j0, int b,
                                                  double *__restrict__ W, int lane, const double *__restrict__ rd) {
  // W (16 x 16, ld 16) <- inverse of the lower-triangular diagonal block A[j0.., j0..];
  // lane c computes column c by column-oriented forward substitution: the
  // dependent chain is one multiply + one FMA per step
  if (lane < b) {
    const int c = lane;
    double x[PIVB_NB];
#pragma unroll
    for (int i = 0; i < PIVB_NB; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < PIVB_NB; ++k) {
      if (k < b) {
        x[k] *= rd[j0 + k];
#pragma unroll
        for (int i = k + 1; i < PIVB_NB; ++i)
          if (i < b) x[i] = fma(-A[(j0 + i) + (j0 + k) * lda], x[k], x[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < PIVB_NB; ++i) W[i + c * PIVB_NB] = (i < b && i >= c) ? x[i] : 0.0;
  }
}

// Shared-memory layout of k_pivot_blk: n padded to a multiple of 16 (the DMMA
// fragments never leave the array; padding is zero), leading dimension
// npad + 4 (= 4 mod 16 doubles: the 8 x 4 A/B and 8 x (2 x 4) C fragment
// patterns of m8n8k4 hit every bank exactly twice, i.e. 2 wavefronts).
__host__ __device__ constexpr int pivb_npad(int n) { return (n + 15) & ~15; }
__host__ __device__ constexpr int pivb_lda(int n) { return pivb_npad(n) + 4; }
__host__ __device__ constexpr size_t pivb_smem_bytes(int n) { return (size_t)pivb_npad(n) * pivb_lda(n) * 8; }

// A fragment (8 x 4, row-major) of the shared array at rows r0.., columns c0..:
// element (g, t); B fragment (4 x 8) of op(X) with X stored row = n-index:
// element X(r0 + g, c0 + t) as B(t, g).  Both are the same load.
__device__ __forceinline__ double frag_ld(const double *A, int lda, int r0, int c0) {
  const int lane = threadIdx.x & 31;
  return A[(r0 + (lane >> 2)) + (c0 + (lane & 3)) * lda];
}

__global__ void __launch_bounds__(512, 1) k_pivot_blk(const PivTask *__restrict__ tasks, int *status) {
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
    if (!pivb_diag_chol(A, lda, j0, b, t.m, rd, lane, lcol)) {
      if (lane == 0) {
        s_fail = 1;
        if (atomicCAS(&status[0], 0, -3) == 0) status[1] = t.node;
      }
      return;
    }
    pivb_diag_inverse(A, lda, j0, b, W, lane, rd);
    __syncwarp();
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
  if (t.Xo) {
    for (int j = warp; j < n; j += nw)
      for (int i = lane; i < n; i += 32) {
        t.Xo[i + (int64_t)j * t.ldxo] = (i >= j) ? A[i + j * lda] : 0.0;
        // Wt(k = i, c = j) = L^{-1}(c, k) d_c (upper triangular)
        t.Wt[i + j * 64] = (i <= j) ? A[j + i * lda] * ((j < t.m) ? 1.0 : -1.0) : 0.0;
      }
    return;
  }
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i < n; i += 32) t.F[i + (int64_t)j * t.ld] = (i >= j) ? A[i + j * lda] : 0.0;
}

// Blocked no-pivot LU of the fused LU-path pivot, same outputs as k_pivot_lu
// (region 0 <- L^{-1}, unit lower; region 1 <- U^{-T}), for n <= PIVLU_MAXN in
// shared memory with 16-column blocks.  LU: per block the diagonal factor by
// one warp (lane = row), the two 16 x 16 triangular inverses, the panels
// L21 = A21 U11^{-1} and U12 = L11^{-1} A12, the trailing A22 -= L21 U12.
// Inverses, last block first: L21 <- -(X22 L21) X11 and U12 <- -Y11 (U12 Y22)
// with X = L^{-1}, Y = U^{-1} of the already inverted trailing parts (scratch
// TL, TU: n x 16 each).  Singular if |u_kk| <= 1e-14 max|A| (as k_pivot_lu).
constexpr int PIVLU_MAXN = 160;
// no-pivot LU of the b x b diagonal block at j0 by one warp, block in registers
// (lane = row; the pivot row's entries by shuffles).  rd[j0 + k] <- 1 / u_kk.
// Returns false when |u_kk| <= tiny (uniform across the warp).
__device__ __forceinline__ bool lu_diag_factor(double *__restrict__ A, int lda, int j0, int b, double tiny,
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

__device__ __forceinline__ void lu_diag_inverses(const double *__restrict__ A, int lda, int j0, int b,
                                                 double *__restrict__ WL, double *__restrict__ WU, int lane,
                                                 const double *__restrict__ rd) {
  // WL = L11^{-1} (unit lower, column c by lane c); WU = U11^{-1} (upper, row c by
  // lane c); both by column-oriented substitution (one FMA on the chain per step)
  if (lane >= b) return;
  const int c = lane;
  double x[PIVB_NB];
#pragma unroll
  for (int i = 0; i < PIVB_NB; ++i) x[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < PIVB_NB; ++k)
    if (k < b) {
#pragma unroll
      for (int i = k + 1; i < PIVB_NB; ++i)
        if (i < b) x[i] = fma(-A[(j0 + i) + (j0 + k) * lda], x[k], x[i]);
    }
#pragma unroll
  for (int i = 0; i < PIVB_NB; ++i) WL[i + c * PIVB_NB] = (i < b && i >= c) ? x[i] : 0.0;
  // y = e_c^T U11^{-1}: y_j = (delta_cj - sum_{k<j} y_k u_kj) / u_jj
#pragma unroll
  for (int j = 0; j < PIVB_NB; ++j) x[j] = (j == c) ? 1.0 : 0.0;
#pragma unroll
  for (int j = 0; j < PIVB_NB; ++j)
    if (j < b) {
      x[j] *= rd[j0 + j];
#pragma unroll
      for (int jj = j + 1; jj < PIVB_NB; ++jj)
        if (jj < b) x[jj] = fma(-x[j], A[(j0 + j) + (j0 + jj) * lda], x[jj]);
    }
#pragma unroll
  for (int j = 0; j < PIVB_NB; ++j) WU[c + j * PIVB_NB] = (j < b && j >= c) ? x[j] : 0.0;
}

__global__ void __launch_bounds__(512, 1) k_pivot_lu_blk(const PivTask *__restrict__ tasks, int *status) {
  // Same shared-memory layout as k_pivot_blk (npad, lda = npad + 4).  Per
  // 16-column block: warp 0 factors the diagonal block (lu_diag_factor) and
  // inverts both triangles (WL = L11^{-1}, WU = U11^{-1}); the panels
  // L21 = A21 WU and U12^T = A12^T WL^T and the trailing A22 -= L21 U12 run on the
  // FP64 tensor cores (m8n8k4 DMMA, 8 x 8 blocks over the warps).  Inverses,
  // last block first (X = L^{-1} strict lower, Y = U^{-1} upper, one array):
  //   P = L21 X11, Q^T = U12^T Y11^T (in place, rows owned by one warp);
  //   X21 = -X22 P, Y12^T = -Y22^T Q^T (DMMA into registers, written after a barrier).
  extern __shared__ double sh[];
  __shared__ double WL[PIVB_NB * PIVB_NB], WU[PIVB_NB * PIVB_NB];
  __shared__ double rd[PIVLU_MAXN + PIVB_NB];   // 1 / u_kk
  __shared__ double urow[PIVB_NB];
  __shared__ int s_fail;
  __shared__ double s_amax[16];
  pdl_trigger();
  const PivTask t = tasks[blockIdx.x];
  pdl_wait();   // task descriptors are static: read before the wait
  const int n = t.m + t.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int npad = pivb_npad(n), lda = pivb_lda(n);
  const int g = lane >> 2, tq = lane & 3;
  double *A = sh;
  double amax = 0;
  for (int j = warp; j < npad; j += nw)
    for (int i = lane; i < npad; i += 32) {
      const double v = (i < n && j < n) ? t.F[i + (int64_t)j * t.ld] : 0.0;
      A[i + j * lda] = v;
      amax = fmax(amax, fabs(v));
    }
  if (tid == 0) s_fail = 0;
  amax = block_max(amax, s_amax);
  const double tiny = 1e-14 * amax;
  // ---------------- blocked LU (no pivoting) ----------------
  for (int j0 = 0; j0 < n; j0 += PIVB_NB) {
    const int b = min(PIVB_NB, n - j0), j1 = j0 + PIVB_NB;
    if (warp == 0) {
      if (!lu_diag_factor(A, lda, j0, b, tiny, rd, lane, urow)) {
        if (lane == 0) {
          s_fail = 1;
          if (atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
        }
      } else {
        lu_diag_inverses(A, lda, j0, b, WL, WU, lane, rd);
      }
    }
    __syncthreads();
    if (s_fail) return;
    const int nrb = (npad - j1) >> 3;
    if (nrb == 0) break;
    // panels: items < nrb are 8-row blocks of L21 = A21 WU; the rest 8-column
    // blocks of U12, computed as U12^T = A12^T WL^T (rows j of U12^T)
    for (int it = warp; it < 2 * nrb; it += nw) {
      const bool lrow = it < nrb;
      const int r0 = j1 + 8 * (lrow ? it : it - nrb);
      double af[4];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4)
        af[k4] = lrow ? A[(r0 + g) + (j0 + 4 * k4 + tq) * lda] : A[(j0 + 4 * k4 + tq) + (r0 + g) * lda];
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int k = 4 * k4 + tq, col = 8 * cb + g;
          const double bv = lrow ? WU[k + col * PIVB_NB] : WL[col + k * PIVB_NB];
          dmma884(c[cb][0], c[cb][1], af[k4], bv);
        }
      __syncwarp();
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = j0 + 8 * cb + 2 * tq + e;
          if (lrow) A[(r0 + g) + cc * lda] = c[cb][e];
          else A[cc + (r0 + g) * lda] = c[cb][e];
        }
    }
    __syncthreads();
    // trailing: A22(ib, jb) -= L21(ib) U12(jb), every block
    for (int q = warp; q < nrb * nrb; q += nw) {
      const int r0 = j1 + 8 * (q / nrb), s0 = j1 + 8 * (q % nrb);
      double c0 = A[(r0 + g) + (s0 + 2 * tq) * lda], c1 = A[(r0 + g) + (s0 + 2 * tq + 1) * lda];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const double av = A[(r0 + g) + (j0 + 4 * k4 + tq) * lda];     // L21(row, k)
        const double bv = -A[(j0 + 4 * k4 + tq) + (s0 + g) * lda];    // -U12(k, col)
        dmma884(c0, c1, av, bv);
      }
      A[(r0 + g) + (s0 + 2 * tq) * lda] = c0;
      A[(r0 + g) + (s0 + 2 * tq + 1) * lda] = c1;
    }
    __syncthreads();
  }
  if (lu_growth(A, lda, n, s_amax, status) > LU_GROWTH_MAX) {   // no pivoting: check the multipliers
    if (tid == 0 && atomicCAS(&status[0], 0, LORASP_NEED_PIVOT) == 0) status[1] = t.node;
    return;
  }
  // ---------------- blocked inverses, last block first ----------------
  constexpr int MAXI = 3;   // items per warp (2 * nrb <= 36 for npad <= 160)
  const int last = ((n - 1) / PIVB_NB) * PIVB_NB;
  for (int j0 = last; j0 >= 0; j0 -= PIVB_NB) {
    const int b = min(PIVB_NB, n - j0), j1 = j0 + PIVB_NB;
    const int nrb = (npad - j1) >> 3;
    if (warp == 0) lu_diag_inverses(A, lda, j0, b, WL, WU, lane, rd);
    __syncthreads();
    // phase 1: P = L21 X11 (rows), Q^T = U12^T Y11^T (rows j of U12^T), in place
    for (int it = warp; it < 2 * nrb; it += nw) {
      const bool lrow = it < nrb;
      const int r0 = j1 + 8 * (lrow ? it : it - nrb);
      double af[4];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4)
        af[k4] = lrow ? A[(r0 + g) + (j0 + 4 * k4 + tq) * lda] : A[(j0 + 4 * k4 + tq) + (r0 + g) * lda];
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int k = 4 * k4 + tq, col = 8 * cb + g;
          const double bv = lrow ? WL[k + col * PIVB_NB] : WU[col + k * PIVB_NB];
          dmma884(c[cb][0], c[cb][1], af[k4], bv);
        }
      __syncwarp();
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = j0 + 8 * cb + 2 * tq + e;
          if (lrow) A[(r0 + g) + cc * lda] = c[cb][e];
          else A[cc + (r0 + g) * lda] = c[cb][e];
        }
    }
    __syncthreads();
    // phase 2: X21 = -X22 P (X22 unit lower), Y12^T = -Y22^T Q^T (Y22 upper)
    double res[MAXI][2][2];
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int it = warp + u * nw;
      if (it >= 2 * nrb) break;
      const bool lrow = it < nrb;
      const int r0 = j1 + 8 * (lrow ? it : it - nrb);
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      for (int k0 = j1; k0 < r0 + 8; k0 += 4) {
        const int row = r0 + g, kc = k0 + tq;
        double av;
        if (lrow) av = (kc < row) ? A[row + kc * lda] : (kc == row ? 1.0 : 0.0);   // X22(row, k)
        else av = (kc <= row) ? A[kc + row * lda] : 0.0;                           // Y22(k, row)
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          const int col = j0 + 8 * cb + g;
          const double bv = lrow ? A[(k0 + tq) + col * lda] : A[col + (k0 + tq) * lda];   // P(k, c) / Q^T(k, c)
          dmma884(c[cb][0], c[cb][1], av, bv);
        }
      }
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int e = 0; e < 2; ++e) res[u][cb][e] = -c[cb][e];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int it = warp + u * nw;
      if (it >= 2 * nrb) break;
      const bool lrow = it < nrb;
      const int r0 = j1 + 8 * (lrow ? it : it - nrb);
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = j0 + 8 * cb + 2 * tq + e;
          const double v = res[u][cb][e];
          if (lrow) A[(r0 + g) + cc * lda] = v;
          else A[cc + (r0 + g) * lda] = v;
        }
    }
    for (int q = tid; q < b * b; q += blockDim.x) {   // X11 strict lower, Y11 upper
      const int i = q % b, c = q / b;
      A[(j0 + i) + (j0 + c) * lda] = (i > c) ? WL[i + c * PIVB_NB] : WU[i + c * PIVB_NB];
    }
    __syncthreads();
  }
  // region 0 <- L^{-1} (unit lower), region 1 <- U^{-T}
  double *R1 = t.F2 ? t.F2 : t.F + (int64_t)t.ld * n;
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i < n; i += 32) {
      t.F[i + (int64_t)j * t.ld] = (i > j) ? A[i + j * lda] : (i == j ? 1.0 : 0.0);
      R1[i + (int64_t)j * t.ld] = (i >= j) ? A[j + i * lda] : 0.0;
    }
}

// -------------------------------------------- blocked pivot (large nodes) ----
// For n = m + r too large for one CTA's shared memory the fused pivot is
// factored by a right-looking blocked signed Cholesky (64-column panels; panel
// and trailing updates are k_gemm2_dmma launches over all large nodes of the
// wave) and inverted by blocked forward substitution into a scratch X.  Each
// diagonal block K11 = L11 D1 L11^T is one k_pivot_blk task (PivTask::Xo):
// X11 = L11^{-1} into the scratch, Wt = L11^{-T} D1 for the panel L21 = K21 Wt.

// ----------------------------------------------------------------- apply ----
// Forward (Alg. 3) and backward (Alg. 4) over the fused records
//   F = [ L^{-1} (n x n) | Z (n x W) ],  Z = L^{-1} C,  C = coupling to T.
// forward:  y = L^{-1} [rhs_s; 0];  rhs_q -= Z_q^T D y           (q in T)
// backward: u = y - Z x_T;  [x_s; x_b] = L^{-T} D u               (P:l.487-495)
struct ApNode {
  const double *F; // record, column-major, leading dimension ld (even):
                   // SPD [L^{-1} | Z];  LU [L^{-1} | U^{-T} | X | Y^T]
  double *y;       // n doubles, kept between the two passes
  int64_t off_s;   // vector offset of Var/RHS(s)
  int64_t zf_off;  // forward coupling (SPD: Z, LU: Y^T)
  int64_t zb_off;  // backward coupling (SPD: Z, LU: X)
  int64_t lb_off;  // backward triangle (SPD: L^{-1}, LU: U^{-T})
  int sym;         // SPD: apply D = diag(I_m, -I_r)
  int m, r, W, ld;
  int seg0, nseg;
  int nsplit;      // split apply: Z column parts (1 = one CTA streams the whole record)
  int64_t upart;   // split apply: offset of the nsplit x n partial backward sums
  int full;        // LU with partial pivoting: region 0 = L^{-1} P is not lower triangular
};
// one CTA of a split wave: Z columns [c0, c1) of node `node` (part p)
struct ApPart {
  int node, c0, c1, p;
};
struct ApSeg {
  int64_t voff;   // vector offset of the target's Var/RHS
  int w, zc;      // width, column offset inside Z
};

// ---- bulk-async (TMA 1D) streaming helpers --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Column-chunk streamer: a node's record F (column-major, ld n) is consumed as
// runs of whole columns [c0, c1) copied into a 2-stage shared-memory ring with
// cp.async.bulk by thread 0; completion through mbarriers.  Chunk c lives in
// stage c & 1; its parity flips every second use.
struct ColStream {
  const double *base;  // first column of the run
  int n, ncol, cc;     // rows, columns in the run, columns per chunk
  double *buf[2];
  uint64_t *bar;       // 2 mbarriers
  __device__ int nchunks() const { return (ncol + cc - 1) / cc; }
  __device__ void issue(int c) const {
    const int c0 = c * cc, c1 = min(ncol, c0 + cc);
    const uint32_t bytes = (uint32_t)((int64_t)(c1 - c0) * n * 8);   // n = ld (even)
    fence_proxy_async();
    mbar_expect_tx(&bar[c & 1], bytes);
    bulk_g2s(buf[c & 1], base + (int64_t)c0 * n, bytes, &bar[c & 1]);
  }
};

// One CTA per node: the node's record streams through shared memory once per
// pass (forward reads L^{-1}[:, :m] and Z, backward reads Z and L^{-1}[:, :m]).
// Column dots out[j] = sum_{k >= (TRI ? j : 0), k < n} col_j[k] x[k] for the
// columns j in [j0, j1) of a staged chunk (column j at buf + (j - j0) ld), with
// G lanes per column (32 / G columns per warp): short columns (the upper
// levels' small n) waste neither lanes nor shuffles on a whole-warp reduction.
template <int G, bool TRI>
__device__ __forceinline__ void ap_col_dots(const double *__restrict__ buf, int ld, int j0, int j1, int n,
                                            const double *__restrict__ x, double *__restrict__ out, int obase) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int CPW = 32 / G;
  const int sub = lane / G, sl = lane % G;
  for (int jb = j0 + warp * CPW; jb < j1; jb += nw * CPW) {
    const int j = jb + sub;
    double sacc = 0.0;
    if (j < j1) {
      const double *col = buf + (int64_t)(j - j0) * ld;
      for (int k = (TRI ? j : 0) + sl; k < n; k += G) sacc = fma(col[k], x[k], sacc);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (sl == 0 && j < j1) out[j - obase] = sacc;
  }
}
template <bool TRI>
__device__ __forceinline__ void ap_col_dots_n(const double *__restrict__ buf, int ld, int j0, int j1, int n,
                                              const double *__restrict__ x, double *__restrict__ out, int obase) {
  if (n <= 64) ap_col_dots<8, TRI>(buf, ld, j0, j1, n, x, out, obase);
  else if (n <= 128) ap_col_dots<16, TRI>(buf, ld, j0, j1, n, x, out, obase);
  else ap_col_dots<32, TRI>(buf, ld, j0, j1, n, x, out, obase);
}
// Row sums acc[i] (+)= sum_{k in [k0, k1), k <= kmax(i)} buf[(k - k0) ld + i] x[k]
// for the rows i < n of a staged chunk: G = 256 / rows-per-group thread groups
// interleave the columns (rows up to 64: 4 groups, up to 128: 2), partial sums
// combined in a fixed order through `part` (>= 256 doubles); SUB: subtract.
// kmax(i) = TRIL ? i : k1 - 1.  Ends with a block barrier.
template <bool SUB>
__device__ __forceinline__ void ap_row_sums(const double *__restrict__ buf, int ld, int k0, int k1, int n, bool tril,
                                            const double *__restrict__ x, double *__restrict__ acc,
                                            double *__restrict__ part) {
  const int tid = threadIdx.x;
  const int G = (n <= 64) ? 4 : (n <= 128 ? 2 : 1);
  if (G == 1) {
    for (int i = tid; i < n; i += blockDim.x) {
      double s0 = 0, s1 = 0;
      const int kl = tril ? min(k1 - 1, i) : k1 - 1;
      int k = k0;
      for (; k + 1 <= kl; k += 2) {
        s0 = fma(buf[(int64_t)(k - k0) * ld + i], x[k], s0);
        s1 = fma(buf[(int64_t)(k + 1 - k0) * ld + i], x[k + 1], s1);
      }
      if (k <= kl) s0 = fma(buf[(int64_t)(k - k0) * ld + i], x[k], s0);
      acc[i] = SUB ? acc[i] - (s0 + s1) : acc[i] + (s0 + s1);
    }
    __syncthreads();
    return;
  }
  const int rpg = blockDim.x / G, g = tid / rpg, i = tid % rpg;
  double s = 0;
  if (i < n) {
    const int kl = tril ? min(k1 - 1, i) : k1 - 1;
    for (int k = k0 + g; k <= kl; k += G) s = fma(buf[(int64_t)(k - k0) * ld + i], x[k], s);
  }
  part[tid] = s;
  __syncthreads();
  if (g == 0 && i < n) {
    double t = part[i];
    for (int q = 1; q < G; ++q) t += part[q * rpg + i];
    acc[i] = SUB ? acc[i] - t : acc[i] + t;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_apply_fwd(const ApNode *__restrict__ nodes,
                                                   const ApSeg *__restrict__ segs,
                                                   double *__restrict__ vec, int chunk_doubles) {
  // PDL: the record (written by the factorization) is fetched before waiting
  // for the previous wave; only the vector depends on it
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) uint64_t bars[2];
  const ApNode nd = nodes[blockIdx.x];
  const int n = nd.m + nd.r;
  if (n == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *stage0 = sh, *stage1 = sh + chunk_doubles;
  double *rhs = stage1 + chunk_doubles;  // m
  double *dy = rhs + nd.m;               // n (accumulates y)
  double *zo = dy + n;                   // W: Z^T D y, written back once at the end
  double *tv = zo + nd.W;                // W: the targets' RHS entries (prefetched)
  double *part = tv + nd.W;              // 256: row-sum partials
  const int ld = nd.ld;
  const int cc = max(1, chunk_doubles / ld);
  const double *Z = nd.F + nd.zf_off;
  const int na = (nd.m + cc - 1) / cc;   // L^{-1}[:, :m] chunks, then Z chunks
  const int nb = (nd.W + cc - 1) / cc;
  const int ntot = na + nb;
  auto issue = [&](int c) {
    const double *src;
    int c0, c1;
    if (c < na) {
      c0 = c * cc;
      c1 = min(nd.m, c0 + cc);
      src = nd.F + (int64_t)c0 * ld;
    } else {
      c0 = (c - na) * cc;
      c1 = min(nd.W, c0 + cc);
      src = Z + (int64_t)c0 * ld;
    }
    const uint32_t bytes = (uint32_t)((int64_t)(c1 - c0) * ld * 8);
    fence_proxy_async();
    mbar_expect_tx(&bars[c & 1], bytes);
    bulk_g2s((c & 1) ? stage1 : stage0, src, bytes, &bars[c & 1]);
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ntot > 0) issue(0);
    if (ntot > 1) issue(1);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = tid; i < nd.m; i += blockDim.x) rhs[i] = vec[nd.off_s + i];
  for (int i = tid; i < n; i += blockDim.x) dy[i] = 0.0;
  for (int sg = 0; sg < nd.nseg; ++sg) {   // the scatter's reads, issued early
    const ApSeg S = segs[nd.seg0 + sg];
    for (int j = tid; j < S.w; j += blockDim.x) tv[S.zc + j] = vec[S.voff + j];
  }
  __syncthreads();
  // ---- y = L^{-1}[:, :m] rhs, then Z^T D y ----
  for (int c = 0; c < ntot; ++c) {
    if (tid == 0 && c >= 1 && c + 1 < ntot) issue(c + 1);   // stage (c+1)&1 freed at the end of c-1
    mbar_wait(&bars[c & 1], (c >> 1) & 1);
    const double *buf = (c & 1) ? stage1 : stage0;
    if (c < na) {
      const int k0 = c * cc, k1 = min(nd.m, k0 + cc);
      ap_row_sums<false>(buf, ld, k0, k1, n, !nd.full, rhs, dy, part);
      if (c == na - 1) {
        for (int i = tid; i < n; i += blockDim.x) {
          const double y = dy[i];
          nd.y[i] = y;
          dy[i] = (i < nd.m || !nd.sym) ? y : -y;
        }
      }
    } else {
      const int j0 = (c - na) * cc, j1 = min(nd.W, j0 + cc);
      ap_col_dots_n<false>(buf, ld, j0, j1, n, dy, zo, 0);
    }
    __syncthreads();   // stage (c & 1) is free for chunk c + 2
  }
  // rhs_q -= Z_q^T D y for every target segment (coalesced; read at the start)
  for (int sg = 0; sg < nd.nseg; ++sg) {
    const ApSeg S = segs[nd.seg0 + sg];
    for (int j = tid; j < S.w; j += blockDim.x) vec[S.voff + j] = tv[S.zc + j] - zo[S.zc + j];
  }
  if (na == 0) {  // m == 0 cannot happen for a recorded node; keep y defined
    for (int i = tid; i < n; i += blockDim.x) nd.y[i] = 0.0;
  }
}

__global__ void __launch_bounds__(256) k_apply_bwd(const ApNode *__restrict__ nodes,
                                                   const ApSeg *__restrict__ segs,
                                                   double *__restrict__ vec, int chunk_doubles) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // PDL: record fetched before the wait
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) uint64_t bars[2];
  const ApNode nd = nodes[blockIdx.x];
  const int n = nd.m + nd.r;
  if (n == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *stage0 = sh, *stage1 = sh + chunk_doubles;
  double *u = stage1 + chunk_doubles;  // n
  double *xt = u + n;                  // W
  double *part = xt + nd.W;            // 256: row-sum partials
  const int ld = nd.ld;
  int cc = max(1, chunk_doubles / ld);
  const double *Z = nd.F + nd.zb_off;
  const double *Lb = nd.F + nd.lb_off;
  const int nb = (nd.W + cc - 1) / cc;     // Z chunks first
  const int na = (nd.m + cc - 1) / cc;     // then L^{-1}[:, :m]
  const int ntot = nb + na;
  auto issue = [&](int c) {
    const double *src;
    int c0, c1;
    if (c < nb) {
      c0 = c * cc;
      c1 = min(nd.W, c0 + cc);
      src = Z + (int64_t)c0 * ld;
    } else {
      c0 = (c - nb) * cc;
      c1 = min(nd.m, c0 + cc);
      src = Lb + (int64_t)c0 * ld;
    }
    uint32_t bytes = (uint32_t)((int64_t)(c1 - c0) * ld * 8);
    fence_proxy_async();
    mbar_expect_tx(&bars[c & 1], bytes);
    bulk_g2s((c & 1) ? stage1 : stage0, src, bytes, &bars[c & 1]);
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ntot > 0) issue(0);
    if (ntot > 1) issue(1);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int sg = 0; sg < nd.nseg; ++sg) {
    const ApSeg S = segs[nd.seg0 + sg];
    for (int j = tid; j < S.w; j += blockDim.x) xt[S.zc + j] = vec[S.voff + j];
  }
  for (int i = tid; i < n; i += blockDim.x) u[i] = nd.y[i];
  __syncthreads();
  for (int c = 0; c < ntot; ++c) {
    if (tid == 0 && c >= 1 && c + 1 < ntot) issue(c + 1);   // stage (c+1)&1 freed at the end of c-1
    mbar_wait(&bars[c & 1], (c >> 1) & 1);
    const double *buf = (c & 1) ? stage1 : stage0;
    if (c < nb) {
      const int j0 = c * cc, j1 = min(nd.W, j0 + cc);
      ap_row_sums<true>(buf, ld, j0, j1, n, false, xt, u, part);
      if (c == nb - 1 && nd.sym) {
        for (int i = nd.m + tid; i < n; i += blockDim.x) u[i] = -u[i];   // D u
      }
    } else {
      if (nb == 0 && c == 0 && nd.sym) {
        for (int i = nd.m + tid; i < n; i += blockDim.x) u[i] = -u[i];
        __syncthreads();
      }
      const int i0 = (c - nb) * cc, i1 = min(nd.m, i0 + cc);
      ap_col_dots_n<true>(buf, ld, i0, i1, n, u, vec + nd.off_s, 0);
    }
    __syncthreads();
  }
}

// ---- dataflow apply (single GPU): one persistent launch per direction ------
// Alg. 3 / Alg. 4 as a dependency graph instead of wave-synchronous launches:
// CTAs claim nodes in elimination order (forward) or its reverse (backward)
// from a global counter and start a node as soon as the nodes it depends on
// have finished (per-node counters: a node's Z^T D y contributions, or its
// targets' x, are complete) instead of waiting for the whole previous wave.
// Forward contributions are not read-modify-written into the targets: each
// node stores Z^T D y in its own slot of `zob`, and the reader subtracts its
// contributions from its RHS in writer (= elimination) order -- the same
// sequence of operations as the wave launches, so the result is bitwise
// theirs.  A node only waits for nodes claimed before it, so the claimed
// node of lowest index can always proceed (no residency assumption).  The
// trailing waves whose few large records are split over CTAs (the wave path's
// split kernels) stay wave launches: the forward pass then ends with flush
// tasks that subtract the dataflow nodes' contributions from those readers'
// RHS (in writer order), and the backward dataflow pass starts after them.
struct ApDf {
  int node;        // the apply node; a flush task (index >= the dataflow nodes) names the reader it updates
  int fin, bin;    // notifications to wait for: forward (distinct writers), backward (distinct targets)
  int c0, nc;      // contributions to this node's RHS, [c0, c0 + nc) of the contribution list (writer order)
  int r0, nr;      // the nodes this node writes into (forward notifications), in dflist
  int w0, nwr;     // the nodes writing into this node (backward notifications), in dflist
  int64_t zo;      // this node's Z^T D y in zob (W doubles)
};
struct ApContrib {
  int64_t src;     // zob offset of the first value
  int off, w;      // offset inside the reader's RHS, width
};
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void df_wait(const int *cnt, int need) {
  if (threadIdx.x == 0)
    while (ld_acquire(cnt) < need) __nanosleep(64);
  __syncthreads();
}
__device__ __forceinline__ void df_notify(int *cnt, const int *list, int k0, int nk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    for (int k = 0; k < nk; ++k) atomicAdd(cnt + list[k0 + k], 1);
  }
}

__global__ void __launch_bounds__(256) k_apply_fwd_df(const ApNode *__restrict__ nodes, const ApDf *__restrict__ dfs,
                                                      const ApContrib *__restrict__ contr, const int *__restrict__ dfl,
                                                      int nnodes, int ntasks, double *__restrict__ vec,
                                                      double *__restrict__ zob, int *cnt, int *work, int chunk_doubles) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ int s_p;
  const int tid = threadIdx.x;
  double *stage0 = sh, *stage1 = sh + chunk_doubles, *rhs = stage1 + chunk_doubles;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t ph = 0;   // phase bit per stage
  for (;;) {
    if (tid == 0) s_p = atomicAdd(work, 1);
    __syncthreads();
    const int p = s_p;
    if (p >= ntasks) break;
    const ApDf df = dfs[p];
    const ApNode nd = nodes[df.node];
    if (p >= nnodes) {   // flush: a wave-launched reader's contributions from the dataflow nodes
      df_wait(cnt + p, df.fin);
      for (int i = tid; i < nd.m; i += blockDim.x) {
        double v = __ldcg(vec + nd.off_s + i);
        bool hit = false;
        for (int c = 0; c < df.nc; ++c) {
          const ApContrib C = contr[df.c0 + c];
          if (i >= C.off && i < C.off + C.w) {
            v -= __ldcg(zob + C.src + (i - C.off));
            hit = true;
          }
        }
        if (hit) vec[nd.off_s + i] = v;
      }
      __syncthreads();
      continue;
    }
    const int n = nd.m + nd.r;
    if (n == 0) {
      df_wait(cnt + p, df.fin);
      df_notify(cnt, dfl, df.r0, df.nr);
      continue;
    }
    double *dy = rhs + nd.m, *part = dy + n;
    const int ld = nd.ld;
    const int cc = max(1, chunk_doubles / ld);
    const double *Z = nd.F + nd.zf_off;
    const int na = (nd.m + cc - 1) / cc, nb = (nd.W + cc - 1) / cc, ntot = na + nb;
    auto issue = [&](int c) {
      const double *src;
      int c0, c1;
      if (c < na) {
        c0 = c * cc;
        c1 = min(nd.m, c0 + cc);
        src = nd.F + (int64_t)c0 * ld;
      } else {
        c0 = (c - na) * cc;
        c1 = min(nd.W, c0 + cc);
        src = Z + (int64_t)c0 * ld;
      }
      const uint32_t bytes = (uint32_t)((int64_t)(c1 - c0) * ld * 8);
      fence_proxy_async();
      mbar_expect_tx(&bars[c & 1], bytes);
      bulk_g2s((c & 1) ? stage1 : stage0, src, bytes, &bars[c & 1]);
    };
    if (tid == 0) {   // the record is static: fetched before the dependencies are met
      if (ntot > 0) issue(0);
      if (ntot > 1) issue(1);
    }
    df_wait(cnt + p, df.fin);
    // RHS = initial entries minus the contributions, in writer order per entry
    for (int i = tid; i < nd.m; i += blockDim.x) {
      double v = __ldcg(vec + nd.off_s + i);
      for (int c = 0; c < df.nc; ++c) {
        const ApContrib C = contr[df.c0 + c];
        if (i >= C.off && i < C.off + C.w) v -= __ldcg(zob + C.src + (i - C.off));
      }
      rhs[i] = v;
    }
    for (int i = tid; i < n; i += blockDim.x) dy[i] = 0.0;
    __syncthreads();
    for (int c = 0; c < ntot; ++c) {
      if (tid == 0 && c >= 1 && c + 1 < ntot) issue(c + 1);
      mbar_wait(&bars[c & 1], (ph >> (c & 1)) & 1);
      ph ^= 1u << (c & 1);
      const double *buf = (c & 1) ? stage1 : stage0;
      if (c < na) {
        const int k0 = c * cc, k1 = min(nd.m, k0 + cc);
        ap_row_sums<false>(buf, ld, k0, k1, n, !nd.full, rhs, dy, part);
        if (c == na - 1) {
          for (int i = tid; i < n; i += blockDim.x) {
            const double y = dy[i];
            nd.y[i] = y;
            dy[i] = (i < nd.m || !nd.sym) ? y : -y;
          }
        }
      } else {
        const int j0 = (c - na) * cc, j1 = min(nd.W, j0 + cc);
        ap_col_dots_n<false>(buf, ld, j0, j1, n, dy, zob + df.zo, 0);
      }
      __syncthreads();
    }
    if (na == 0)
      for (int i = tid; i < n; i += blockDim.x) nd.y[i] = 0.0;
    df_notify(cnt, dfl, df.r0, df.nr);
  }
}

__global__ void __launch_bounds__(256) k_apply_bwd_df(const ApNode *__restrict__ nodes, const ApDf *__restrict__ dfs,
                                                      const ApSeg *__restrict__ segs, const int *__restrict__ dfl,
                                                      int nnodes, double *__restrict__ vec, int *cnt, int *work,
                                                      int chunk_doubles) {
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ int s_p;
  const int tid = threadIdx.x;
  double *stage0 = sh, *stage1 = sh + chunk_doubles, *u = stage1 + chunk_doubles;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t ph = 0;
  for (;;) {
    if (tid == 0) s_p = atomicAdd(work, 1);
    __syncthreads();
    const int p = nnodes - 1 - s_p;
    if (p < 0) break;
    const ApDf df = dfs[p];
    const ApNode nd = nodes[df.node];
    const int n = nd.m + nd.r;
    if (n == 0) {
      df_wait(cnt + p, df.bin);
      df_notify(cnt, dfl, df.w0, df.nwr);
      continue;
    }
    double *xt = u + n, *part = xt + nd.W;
    const int ld = nd.ld;
    const int cc = max(1, chunk_doubles / ld);
    const double *Z = nd.F + nd.zb_off, *Lb = nd.F + nd.lb_off;
    const int nb = (nd.W + cc - 1) / cc, na = (nd.m + cc - 1) / cc, ntot = nb + na;
    auto issue = [&](int c) {
      const double *src;
      int c0, c1;
      if (c < nb) {
        c0 = c * cc;
        c1 = min(nd.W, c0 + cc);
        src = Z + (int64_t)c0 * ld;
      } else {
        c0 = (c - nb) * cc;
        c1 = min(nd.m, c0 + cc);
        src = Lb + (int64_t)c0 * ld;
      }
      const uint32_t bytes = (uint32_t)((int64_t)(c1 - c0) * ld * 8);
      fence_proxy_async();
      mbar_expect_tx(&bars[c & 1], bytes);
      bulk_g2s((c & 1) ? stage1 : stage0, src, bytes, &bars[c & 1]);
    };
    if (tid == 0) {
      if (ntot > 0) issue(0);
      if (ntot > 1) issue(1);
    }
    df_wait(cnt + p, df.bin);
    for (int sg = 0; sg < nd.nseg; ++sg) {
      const ApSeg S = segs[nd.seg0 + sg];
      for (int j = tid; j < S.w; j += blockDim.x) xt[S.zc + j] = __ldcg(vec + S.voff + j);
    }
    for (int i = tid; i < n; i += blockDim.x) u[i] = __ldcg(nd.y + i);
    __syncthreads();
    for (int c = 0; c < ntot; ++c) {
      if (tid == 0 && c >= 1 && c + 1 < ntot) issue(c + 1);
      mbar_wait(&bars[c & 1], (ph >> (c & 1)) & 1);
      ph ^= 1u << (c & 1);
      const double *buf = (c & 1) ? stage1 : stage0;
      if (c < nb) {
        const int j0 = c * cc, j1 = min(nd.W, j0 + cc);
        ap_row_sums<true>(buf, ld, j0, j1, n, false, xt, u, part);
        if (c == nb - 1 && nd.sym)
          for (int i = nd.m + tid; i < n; i += blockDim.x) u[i] = -u[i];   // D u
      } else {
        if (nb == 0 && c == 0 && nd.sym) {
          for (int i = nd.m + tid; i < n; i += blockDim.x) u[i] = -u[i];
          __syncthreads();
        }
        const int i0 = (c - nb) * cc, i1 = min(nd.m, i0 + cc);
        ap_col_dots_n<true>(buf, ld, i0, i1, n, u, vec + nd.off_s, 0);
      }
      __syncthreads();
    }
    df_notify(cnt, dfl, df.w0, df.nwr);
  }
}

// ---- split apply (waves with few, large records) --------------------------
// The fused kernels stream a node's whole record with one CTA; for the upper
// levels (few nodes per wave, records of MBs) the Z columns are split over
// CTAs instead.  Forward: k_apply_fwd_y (y = L^{-1}[:, :m] rhs, one CTA per
// node) then k_apply_fwd_z (zo = Z^T D y for a column slice, scattered into the
// targets; slices own disjoint target entries).  Backward: k_apply_bwd_z
// (partial Z x_T per slice into scratch) then k_apply_bwd_l (u = y - sum of
// the partials in slice order, D u, x_s = L^{-T} u): deterministic.
// Split wave, forward: rows [P.c0, P.c1) (<= 64) of y = L^{-1}[:, :m] rhs for node
// P.node, one CTA per row slab: 64 rows x 4 interleaved column groups (reads
// coalesced down each column), the four partial sums combined in shared memory.
__global__ void __launch_bounds__(256) k_apply_fwd_y(const ApNode *__restrict__ nodes, const ApPart *__restrict__ parts,
                                                     double *__restrict__ vec) {
  pdl_enter();
  extern __shared__ __align__(16) double sh[];
  const ApPart P = parts[blockIdx.x];
  const ApNode nd = nodes[P.node];
  const int n = nd.m + nd.r;
  if (n == 0) return;
  double *rhs = sh, *red = sh + nd.m;   // m | 4 x 64 partial sums
  for (int i = threadIdx.x; i < nd.m; i += blockDim.x) rhs[i] = vec[nd.off_s + i];
  __syncthreads();
  const int row = threadIdx.x & 63, grp = threadIdx.x >> 6, i = P.c0 + row;
  double s0 = 0, s1 = 0;
  if (i < P.c1) {
    const int kl = nd.full ? nd.m - 1 : min(nd.m - 1, i);
    const double *Fi = nd.F + i;
    int k = grp;
    for (; k + 4 <= kl; k += 8) {
      s0 = fma(Fi[(int64_t)k * nd.ld], rhs[k], s0);
      s1 = fma(Fi[(int64_t)(k + 4) * nd.ld], rhs[k + 4], s1);
    }
    for (; k <= kl; k += 4) s0 = fma(Fi[(int64_t)k * nd.ld], rhs[k], s0);
  }
  red[grp * 64 + row] = s0 + s1;
  __syncthreads();
  if (grp == 0 && i < P.c1) nd.y[i] = (red[row] + red[64 + row]) + (red[128 + row] + red[192 + row]);
}

__global__ void __launch_bounds__(256) k_apply_fwd_z(const ApNode *__restrict__ nodes, const ApPart *__restrict__ parts,
                                                     const ApSeg *__restrict__ segs, double *__restrict__ vec,
                                                     int chunk_doubles) {
  pdl_enter();
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) uint64_t bars[2];
  const ApPart P = parts[blockIdx.x];
  const ApNode nd = nodes[P.node];
  const int n = nd.m + nd.r, ncol = P.c1 - P.c0;
  if (n == 0 || ncol <= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *stage0 = sh, *stage1 = sh + chunk_doubles, *dy = stage1 + chunk_doubles, *zo = dy + n;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < n; i += blockDim.x) {
    const double y = nd.y[i];
    dy[i] = (i < nd.m || !nd.sym) ? y : -y;
  }
  __syncthreads();
  const int ld = nd.ld;
  const int cc = max(1, chunk_doubles / ld);
  ColStream Bz{nd.F + nd.zf_off + (int64_t)P.c0 * ld, ld, ncol, cc, {stage0, stage1}, bars};
  const int nb = Bz.nchunks();
  if (tid == 0) Bz.issue(0);
  for (int c = 0; c < nb; ++c) {
    if (tid == 0 && c + 1 < nb) Bz.issue(c + 1);
    mbar_wait(&bars[c & 1], (c >> 1) & 1);
    const double *buf = (c & 1) ? stage1 : stage0;
    const int j0 = c * cc, j1 = min(ncol, j0 + cc);
    for (int j = j0 + warp; j < j1; j += nw) {
      const double *col = buf + (int64_t)(j - j0) * ld;
      double sacc = 0;
      for (int k = lane; k < n; k += 32) sacc = fma(col[k], dy[k], sacc);
      sacc = warp_sum(sacc);
      if (lane == 0) zo[j] = sacc;
    }
    __syncthreads();
  }
  // scatter the slice: Z column P.c0 + j belongs to the segment covering it
  for (int sg = 0; sg < nd.nseg; ++sg) {
    const ApSeg S = segs[nd.seg0 + sg];
    const int a = max(S.zc, P.c0), b = min(S.zc + S.w, P.c1);
    for (int j = a + tid; j < b; j += blockDim.x) vec[S.voff + (j - S.zc)] -= zo[j - P.c0];
  }
}

__global__ void __launch_bounds__(256) k_apply_bwd_z(const ApNode *__restrict__ nodes, const ApPart *__restrict__ parts,
                                                     const ApSeg *__restrict__ segs, const double *__restrict__ vec,
                                                     double *__restrict__ upart, int chunk_doubles) {
  pdl_enter();
  extern __shared__ __align__(16) double sh[];
  __shared__ __align__(8) uint64_t bars[2];
  const ApPart P = parts[blockIdx.x];
  const ApNode nd = nodes[P.node];
  const int n = nd.m + nd.r, ncol = P.c1 - P.c0;
  if (n == 0) return;
  const int tid = threadIdx.x;
  double *stage0 = sh, *stage1 = sh + chunk_doubles, *xt = stage1 + chunk_doubles, *u = xt + ncol;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int sg = 0; sg < nd.nseg; ++sg) {
    const ApSeg S = segs[nd.seg0 + sg];
    const int a = max(S.zc, P.c0), b = min(S.zc + S.w, P.c1);
    for (int j = a + tid; j < b; j += blockDim.x) xt[j - P.c0] = vec[S.voff + (j - S.zc)];
  }
  for (int i = tid; i < n; i += blockDim.x) u[i] = 0.0;
  __syncthreads();
  const int ld = nd.ld;
  const int cc = max(1, chunk_doubles / ld);
  ColStream Bz{nd.F + nd.zb_off + (int64_t)P.c0 * ld, ld, ncol, cc, {stage0, stage1}, bars};
  const int nb = ncol > 0 ? Bz.nchunks() : 0;
  if (tid == 0 && nb > 0) Bz.issue(0);
  for (int c = 0; c < nb; ++c) {
    if (tid == 0 && c + 1 < nb) Bz.issue(c + 1);
    mbar_wait(&bars[c & 1], (c >> 1) & 1);
    const double *buf = (c & 1) ? stage1 : stage0;
    const int j0 = c * cc, j1 = min(ncol, j0 + cc);
    for (int i = tid; i < n; i += blockDim.x) {
      double s0 = 0, s1 = 0;
      int j = j0;
      for (; j + 1 < j1; j += 2) {
        s0 = fma(buf[(int64_t)(j - j0) * ld + i], xt[j], s0);
        s1 = fma(buf[(int64_t)(j + 1 - j0) * ld + i], xt[j + 1], s1);
      }
      if (j < j1) s0 = fma(buf[(int64_t)(j - j0) * ld + i], xt[j], s0);
      u[i] += s0 + s1;
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) upart[nd.upart + (int64_t)P.p * n + i] = u[i];
}

// Split wave, backward: x_i = (L^{-1})^T D u for the columns i in [P.c0, P.c1)
// of node P.node (u = y - the Z-part sums), one CTA per column slab, a warp
// per column (each CTA forms u itself: n x nsplit loads).
__global__ void __launch_bounds__(256) k_apply_bwd_l(const ApNode *__restrict__ nodes, const ApPart *__restrict__ parts,
                                                     const double *__restrict__ upart, double *__restrict__ vec) {
  pdl_enter();
  extern __shared__ __align__(16) double sh[];
  const ApPart P = parts[blockIdx.x];
  const ApNode nd = nodes[P.node];
  const int n = nd.m + nd.r;
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double *u = sh;
  for (int i = tid + P.c0; i < n; i += blockDim.x) {   // rows >= c0 are all the columns read
    double acc = nd.y[i];
    for (int p = 0; p < nd.nsplit; ++p) acc -= upart[nd.upart + (int64_t)p * n + i];
    u[i] = (i < nd.m || !nd.sym) ? acc : -acc;   // D u
  }
  __syncthreads();
  const double *Lb = nd.F + nd.lb_off;
  for (int i = P.c0 + warp; i < P.c1; i += nw) {
    const double *col = Lb + (int64_t)i * nd.ld;
    double sacc = 0;
    for (int k = i + lane; k < n; k += 32) sacc = fma(col[k], u[k], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) vec[nd.off_s + i] = sacc;
  }
}

__global__ void k_set_rhs(const double *__restrict__ b, const int64_t *__restrict__ perm, int64_t n,
                          double *__restrict__ vec) {
  pdl_enter();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    vec[perm[q]] = b[q];
}
__global__ void k_get_x(const double *__restrict__ vec, const int64_t *__restrict__ perm, int64_t n,
                        double *__restrict__ x) {
  pdl_enter();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    x[q] = vec[perm[q]];
}

// ---------------------------------------------------------------- Krylov ----
__global__ void k_spmv(int64_t n, const int64_t *__restrict__ rp, const int64_t *__restrict__ ci,
                       const double *__restrict__ va, const double *__restrict__ x,
                       double *__restrict__ y) {
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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
// PCG with device-resident scalars (one host round trip per iteration):
// x += a p, r -= a q with a = rz / pq; a breakdown (pq <= 0 or rz <= 0,
// reading Z24) leaves x, r unchanged and raises *flag
__global__ void k_pcg_update(int64_t n, const double *__restrict__ s_rz, const double *__restrict__ s_pq,
                             const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ x,
                             double *__restrict__ r, double *__restrict__ flag) {
  pdl_enter();
  const double rz = *s_rz, pq = *s_pq;
  const bool ok = (pq > 0) && (rz > 0);
  const double a = ok ? rz / pq : 0.0;
  if (!ok && blockIdx.x == 0 && threadIdx.x == 0) *flag = 1.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = a * p[i] + x[i];
    r[i] = -a * q[i] + r[i];
  }
}
// p = z + (rz_new / rz_old) p
__global__ void k_pcg_dir(int64_t n, const double *__restrict__ s_new, const double *__restrict__ s_old,
                          const double *__restrict__ z, double *__restrict__ p) {
  pdl_enter();
  const double beta = *s_new / *s_old;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
// y += sgn * (*s) * x with the scalar on the device (GMRES Gram-Schmidt step)
__global__ void k_axpy_dev(int64_t n, const double *__restrict__ s, double sgn, const double *__restrict__ x,
                           double *__restrict__ y) {
  pdl_enter();
  const double a = sgn * *s;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + y[i];
}
// y = a*x + b*y
__global__ void k_axpby(int64_t n, double a, const double *__restrict__ x, double b,
                        double *__restrict__ y) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (b == 0.0) ? a * x[i] : a * x[i] + b * y[i];   // b = 0: y is output only (may be uninitialised)
}
// z = x - y
__global__ void k_sub(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                      double *__restrict__ z) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = x[i] - y[i];
}

}  // namespace lorasp
