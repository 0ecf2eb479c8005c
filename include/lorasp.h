/*
 * liblorasp — B200-native (sm_100a) LoRaSp level sweep: the hierarchical
 * low-rank approximate LU of a sparse matrix of arxiv 1510.07363
 * ("LoRaSp"), used as a direct solver or as a Krylov preconditioner.
 *
 * C ABI: plain pointers and sizes, no torch / C++ types.  Every entry point
 * returns an lorasp_status (0 = OK, > 0 soft, < 0 hard error); the message of
 * the last error is available from lorasp_last_error().  Hard errors leave the
 * handle valid but unfactored.
 *
 * Pointers that carry numeric data (values, b, x) may be HOST or DEVICE
 * pointers: the library inspects them with cudaPointerGetAttributes and copies
 * host buffers through its own device staging (the "e2e" path).  Device
 * pointers must live on the handle's device.  Caller-owned memory is only
 * borrowed for the duration of the call; the library owns everything it
 * allocates and frees it in lorasp_destroy().
 *
 * Citations: "P:l.N" = line N of the paper text.
 */
#ifndef LORASP_H
#define LORASP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lorasp_ctx *lorasp_handle;  /* opaque, owned by the library */

typedef enum {
  LORASP_OK = 0,
  LORASP_NOT_CONVERGED = 1,     /* soft: Krylov hit max_it; x holds the last iterate      */
  LORASP_E_ARG = -1,            /* bad argument (null pointer, size, flag)                */
  LORASP_E_PATTERN = -2,        /* pattern not usable (asymmetric structure, bad CSR)     */
  LORASP_E_SINGULAR_PIVOT = -3, /* a pivot's signed Cholesky failed (node in last_error)  */
  LORASP_E_EIG_NOCONV = -4,     /* Jacobi eigen-solver did not converge                   */
  LORASP_E_CUDA = -5,           /* CUDA runtime error                                     */
  LORASP_E_OOM = -6,            /* device allocation failed                               */
  LORASP_E_NCCL = -7,           /* reserved for the multi-GPU exchange                    */
  LORASP_E_STATE = -8           /* call out of order (e.g. apply before factor)           */
} lorasp_status;

/* analyze flags */
#define LORASP_SPD            0x1u  /* symmetric input: symmetric block store, SPD path  */
#define LORASP_ORDER_NATURAL  0x2u  /* ascending cluster order, one node per wave (debug:
                                       the paper's literal Alg. 1 loop, P:l.281)         */
#define LORASP_RRQR           0x4u  /* Compress with rank-revealing (column-pivoted) QR
                                       instead of the SVD (P:l.616, P:l.840; SURVEY 8(f)
                                       f1): keep the leading k with |R_kk| >= eps |R_00|;
                                       nodes with m <= 512 (LORASP_E_ARG beyond)          */
#define LORASP_ALGEBRAIC      0x10u /* nested partitionings from the graph of A alone (BFS
                                       level-structure bisection; coords
                                       may be NULL and dim is ignored)                    */
#define LORASP_FROBENIUS      0x20u /* truncation by the Frobenius rule Eq. curOff6
                                       (P:l.756-761): keep the smallest k
                                       with ||B - U_k S_k V_k^T||_F < eps ||all levels
                                       below||_F, the denominator = every super-node block
                                       of this and the deeper levels right after
                                       MergeRedNodes (reading F2); SVD only    */

/* Krylov methods for lorasp_krylov_ex */
#define LORASP_CG     0
#define LORASP_GMRES  1

/*
 * lorasp_analyze — symbolic phase (host only; no device work).
 *   Builds the nested partitionings P_0..P_depth by recursive coordinate
 *   bisection (Def. nested partitionings, P:l.214-216), the quotient graphs of
 *   A at every level (Def. adjacency graph P:l.73-76, adjacent clusters
 *   P:l.247-249), a distance-2 colouring per level (the order within a level
 *   is free, P:l.843), and replays Alg. 1 (P:l.265-289) symbolically: per
 *   super-node the well-separated partners, the neighbours it is eliminated
 *   against and every block that fill creates (Theorem, P:l.515-521).
 *
 *   n         number of unknowns (> 0)
 *   row_ptr   host, n+1 int64, CSR row pointers of A (row_ptr[0] = 0)
 *   col_idx   host, nnz int64, column indices, sorted within each row; the
 *             pattern must be structurally symmetric (else LORASP_E_PATTERN)
 *   dim       coordinate dimension (1..3)
 *   coords    host, n*dim float64, row-major point coordinates
 *   leaf_size target dofs per leaf red cluster (used when depth <= 0)
 *   depth     H-tree depth l; <= 0 means round(log2(n / leaf_size))
 *   eps       truncation threshold of Eq. cutOff1 (P:l.580-584): keep
 *             sigma_k >= eps * sigma_0; eps = 0 keeps everything (exact)
 *   flags     LORASP_SPD (symmetric input; else the general LU path) |
 *             LORASP_ORDER_NATURAL | LORASP_RRQR | LORASP_ALGEBRAIC
 *   device    CUDA device ordinal the handle will use
 *   out       receives the handle
 *   The pattern and coordinates are copied; the caller keeps ownership.
 */
int lorasp_analyze(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                   int dim, const double *coords, int leaf_size, int depth,
                   double eps, unsigned flags, int device, lorasp_handle *out);

/*
 * lorasp_factor — numeric phase: Alg. 1 (P:l.265-289) on the device.
 *   values  nnz float64 in the CSR order given to analyze (host or device).
 *   Per level: MergeRedNodes (P:l.295-313); per distance-2 colour wave:
 *   Compress (P:l.319-394: batched Gram + symmetric eigen-solver, rank
 *   sigma_k >= eps sigma_0, R_k = A_k V, five edge rules) and the fused
 *   elimination of s and b (P:l.396-399, P:l.101-106).  Re-callable with new
 *   values on the same pattern.  Returns LORASP_E_SINGULAR_PIVOT /
 *   LORASP_E_EIG_NOCONV on numerical failure.
 *   Scheduling (results identical either way): the sweep runs on a
 *   high-priority library stream ordered after the handle's stream and the
 *   call returns synchronised.  The first factorization synchronises once per
 *   compress wave (the ranks size what follows); later calls enqueue every wave
 *   with the previous call's ranks, verify the device ranks after the sweep and
 *   redo the synchronised sweep on a mismatch (stats: schedule_rank_predicted,
 *   rank_prediction_hits / _misses; LORASP_NO_REPLAY=1 disables).
 */
int lorasp_factor(lorasp_handle h, const double *values);

/*
 * lorasp_apply — x = Ã b: Alg. 2-4 (P:l.401-500), forward and backward
 *   substitution over the frozen factors in elimination order.
 *   b, x: n float64 (host or device, both of the same kind); x must not alias b.
 */
int lorasp_apply(lorasp_handle h, const double *b, double *x);

/*
 * lorasp_gmres — right-preconditioned GMRES(50) with Ã (P:l.651-669):
 *   x (in: ignored, x0 = 0; out: solution) until ||b - A x|| / ||b|| <= tol
 *   or 500 iterations (LORASP_NOT_CONVERGED).
 */
int lorasp_gmres(lorasp_handle h, const double *b, double *x, double tol);

/*
 * lorasp_krylov_ex — the full form: method LORASP_CG (preconditioned CG,
 *   P:l.652) or LORASP_GMRES; restart (GMRES, <= 1000; <= 0 means 50), max_it; outputs the number of
 *   iterations (A-products) and the final true relative residual
 *   ||b - A x||_2 / ||b||_2 (Eq. accres, P:l.585-589).  iters / relres may be NULL.
 */
int lorasp_krylov_ex(lorasp_handle h, const double *b, double *x, double tol,
                     int method, int restart, int max_it, int *iters, double *relres);

/*
 * lorasp_paper_residual — the paper's preconditioned residual, Eq. GMRES_residual
 *   (P:l.665-669): *out = ||Ã b - Ã A x||_2 / ||Ã b||_2, computed on the device
 *   (SpMV with the values of the last lorasp_factor, two applications of Ã).
 *   b, x: n float64, host or device (both of the same kind); out: host double.
 *   LORASP_E_STATE before a successful factorization.
 */
int lorasp_paper_residual(lorasp_handle h, const double *b, const double *x, double *out);

/* Use an existing cudaStream_t (passed as void*) for all device work; NULL = default. */
int lorasp_set_stream(lorasp_handle h, void *cuda_stream);

/*
 * Distributed factorization over `world` ranks (one process / handle per GPU),
 * the subtree partition of SURVEY 8(e) (P:l.55: the tree's subtrees are
 * independent up to the separator couplings, P:l.843: distributed memory).
 *   world   power of two with 2^(depth-1) >= world; rank in [0, world).
 *   Owner of level-i super-node c (and of its black node): c >> (i - 1 - log2
 *   world) when i - 1 >= log2 world (the subtree of level-(log2 world + 1)
 *   node g belongs to rank g), else rank 0 (the top levels).
 *   Every rank runs the same host schedule (identical plan, ranks and record
 *   layout) and launches only the tasks of the nodes it owns.  Exchange points
 *   go through `fn`:
 *     after Compress, the ranks of the wave's nodes (and the status flags):
 *       LORASP_COLL_MAXINT — elementwise max over ranks of the first nbytes/4
 *       int32 of the send buffer, in place (non-owned entries are 0);
 *     after the Schur updates (neighbour push): every block a rank wrote goes
 *       only to the ranks that read or update it later (the owners of the
 *       nodes whose plan references it, and the readers of the next level's
 *       block it is merged into); factor records never leave their owner:
 *       LORASP_COLL_ALLTOALLV — rank q's send holds, back to back for p = 0..
 *       world-1, counts[q][p] bytes for rank p; rank p's recv receives, back to
 *       back for q = 0.., counts[q][p] bytes from rank q (lorasp_dist_counts
 *       gives the world x world byte matrix, [q * world + p]);
 *     in the distributed apply, after every colour wave, the vector segments
 *       written there (tiny):
 *       LORASP_COLL_ALLGATHER — rank q's send[0, nbytes) lands in every rank's
 *       recv[q * nbytes, (q + 1) * nbytes).
 *   LORASP_COLL_RESERVE asks for send >= nbytes and recv >= world * nbytes
 *   bytes of device memory; the callback registers them with
 *   lorasp_set_dist_buffers before returning.  The engine synchronises its
 *   stream before every call; the callback returns with the transfer complete
 *   (0 = OK, anything else aborts the factorization with LORASP_E_CUDA).
 *   Distance-2 colouring makes the blocks written in one wave disjoint across
 *   nodes, so every rank's blocks and its own records equal the G = 1 ones bit
 *   for bit.  lorasp_apply / lorasp_krylov_ex are collective in this mode (every
 *   rank calls them): each rank applies its own nodes (see lorasp_set_dist_nccl).
 *   Rank-predicted replay and split pivots are off in this mode.  world <= 32.
 *   world = 1 (or fn = NULL) switches back to the single-GPU sweep.
 */
typedef enum {
  LORASP_COLL_ALLGATHER = 0, LORASP_COLL_MAXINT = 1, LORASP_COLL_RESERVE = 2, LORASP_COLL_ALLTOALLV = 3
} lorasp_coll_kind;
typedef int (*lorasp_coll_fn)(void *user, int kind, int64_t nbytes);
int lorasp_set_dist(lorasp_handle h, int rank, int world, lorasp_coll_fn fn, void *user);
/* byte matrix of the current LORASP_COLL_ALLTOALLV ([src * world + dst]); returns world^2 */
int lorasp_dist_counts(lorasp_handle h, int64_t *counts, int cap);

/*
 * Library-owned communicator (SURVEY 8(b) `comm`): the same distributed mode
 * with the per-wave collectives issued by the library itself through NCCL on
 * its stream (ncclAllGather / ncclAllReduce(max) over library-owned device
 * buffers), no callback.  lorasp_nccl_unique_id fills 128 bytes on one rank;
 * the caller distributes them (any channel); every rank then calls
 * lorasp_set_dist_nccl with its rank, the world size (a power of two) and the
 * same id.  NCCL is resolved at run time (the libnccl.so.2 already loaded, else
 * the system one); LORASP_E_NCCL when unavailable or on an NCCL error.
 * In distributed mode the factor records stay on their owner and lorasp_apply /
 * lorasp_krylov_ex run the apply distributed: each rank applies its own nodes,
 * and after every colour wave the vector segments written there are exchanged
 * (every rank must call them; the Krylov vectors are replicated).
 */
int lorasp_nccl_unique_id(void *id_out);
int lorasp_set_dist_nccl(lorasp_handle h, int rank, int world, const void *unique_id);
/* NCCL plumbing check on one device (1-rank communicator, all-gather + max-reduce of n ints). */
int lorasp_test_nccl(int device, int n);
/* Device buffers (owned by the caller) for the exchanges; capacity in bytes
 * (send_cap >= the reserve request, recv_cap >= world times it). */
int lorasp_set_dist_buffers(lorasp_handle h, void *send, int64_t send_cap, void *recv, int64_t recv_cap);
/* Owner rank of level-`level` super-node c under the partition above (host only). */
int lorasp_dist_owner(int level, int c, int world);

/* Structure queries (valid after analyze): depth l and, for level i (1..l),
 * the number of clusters 2^(i-1) and the processing order of those clusters
 * (order[k] = cluster processed k-th) and its colour waves (wave[c]). */
int lorasp_get_depth(lorasp_handle h, int *depth);
int lorasp_get_level_order(lorasp_handle h, int level, int *order, int *wave, int cap);
/* Per-node edge counts of the symbolic Alg. 1 replay (valid after analyze, host
 * only): partners[c] = number of well-separated super-nodes s_c is compressed
 * against (distance 2, the kappa_2 of Lemma sparse / Theorem, P:l.527-542) and
 * n1[c] = number of uneliminated neighbours at its elimination (distance 1, the
 * kappa_1 edges), counting its own redundant node b when s_c was compressed.  Either pointer may be NULL; cap >= 2^(level-1). */
int lorasp_get_node_counts(lorasp_handle h, int level, int *partners, int *n1, int cap);

/* Numeric queries (valid after factor): per-node retained rank r of s_c^[i]
 * (c = 0..2^(i-1)-1), and per-level super-node sizes m_c.  lorasp_get_stats'
 * "levels" entries summarise them as the paper's FactorStats (P:l.527-558,
 * P:l.729-733): d_max (= d_i) and d_avg, rank_avg, compression_ratio =
 * <rank>_l / <super-node size>_l over the compressed super-nodes, kappa1 /
 * kappa2 (max of the counts above); top level: alpha_hat = max over i < l of
 * (d_i / d_l)^(1/(l-i)) (the growth condition d_i <= alpha^(l-i) d_l checked
 * post hoc, a diagnostic). */
int lorasp_get_ranks(lorasp_handle h, int level, int *ranks, int cap);
int lorasp_get_sizes(lorasp_handle h, int level, int *sizes, int cap);

/* JSON statistics (ranks per level, algorithmic flops, phase times, bytes)
 * into buf (NUL-terminated, truncated to cap). Returns the full length needed
 * through *len if len != NULL. */
int lorasp_get_stats(lorasp_handle h, char *buf, size_t cap, size_t *len);

/* Per-kernel-class CUDA-event timing on the handle's stream.  enable is a
 * bitmask of kernel classes (bit c = the class with "class": c in the stats
 * JSON; -1 = all); nonzero resets and starts accumulating (ms, launches,
 * algorithmic flops and bytes per class, reported under "kernels" by
 * lorasp_get_stats); 0 stops.  Each timed launch costs two event records. */
int lorasp_set_timing(lorasp_handle h, int enable);

/* Number of kernel launches issued by the last factor / apply / krylov call. */
int lorasp_get_launch_count(lorasp_handle h, int64_t *factor_launches,
                            int64_t *apply_launches, int64_t *krylov_launches);

/*
 * lorasp_test_gemm — kernel comparison hook (north_star item 3: FP64 tensor
 *   cores only for block shapes where they beat the FMA path).  Runs `reps`
 *   independent copies of C = op(A) op(B) (one launch, like a wave of equal
 *   GEMMs) through the DFMA tile kernel (variant 0) or the DMMA one (variant 1);
 *   *ms = best CUDA-event time of one launch over 3 timed launches.  Host
 *   buffers: A M x K (ld M) or, ta != 0, K x M (ld K); B K x N (ld K) or, tb,
 *   N x K (ld N); C M x N (ld M) receives the first copy's product.
 */
int lorasp_test_gemm(int device, int variant, int M, int N, int K, int ta, int tb, int reps,
                     const double *A, const double *B, double *C, double *ms);

/*
 * Kernel-level test hooks (host buffers, run on `device`, synchronous).
 * lorasp_test_eig: the Compress eigen-solver on one symmetric PSD Gram matrix
 *   G (m x m, column-major): sigma (m, descending sqrt-eigenvalues), rank
 *   r = #{sigma_k >= eps sigma_0}, V (m x r, column-major) the leading
 *   eigenvectors (P:l.333-359, Eq. cutOff1).
 * lorasp_test_pivot: the fused (s, b) pivot kernel on K = [[S, V], [V^T, 0]]
 *   (n = m + r, column-major, lower triangle read): overwrites K with L^{-1}
 *   where K = L diag(I_m, -I_r) L^T.  Returns LORASP_E_SINGULAR_PIVOT on failure.
 */
int lorasp_test_eig(int device, const double *G, int m, double eps, double *V, double *sigma, int *rank);
int lorasp_test_pivot(int device, double *K, int m, int r);

const char *lorasp_last_error(lorasp_handle h);
void lorasp_destroy(lorasp_handle h);

#ifdef __cplusplus
}
#endif
#endif /* LORASP_H */
