/*
 * prrp_b200.h — C ABI of the B200 (sm_100a) LU_PRRP / CALU_PRRP library.
 *
 * Drop-in boundary for the reference package `prrp` (arXiv 1208.2451
 * reference, /root/reference/pkg/src/prrp).  The reference is pure Python, so
 * its "FFI" is its public Python API; each entry point below replaces the
 * numpy work behind one of those functions (file:line cited per function).
 * The Python mirror package `paper_1208_2451_b200` binds these with ctypes
 * (INTEGRATION.md shows the binding a maintainer of the reference would add).
 *
 * Conventions
 *  - All matrix pointers are DEVICE pointers to float64.  The factorization
 *    matrix is ROW-MAJOR, element (i, j) at A[i*lda + j], lda >= n, lda even
 *    (16-byte row pitch for the TMA descriptors).  The result is stored in
 *    place as the packed L\U of the reference's BlockLUFactors: unit lower L
 *    strictly below the diagonal, U on and above it (luprrp.py:81-87 keeps
 *    them as separate arrays; the Python shim splits them).
 *  - perm is a DEVICE int64 array of length m: row i of the factored matrix
 *    is row perm[i] of the input (matcore.apply_row_perm, matcore.py:152-159).
 *  - Small outputs (stats, error record, swap counts) are HOST pointers;
 *    the call synchronizes the stream before returning them.
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy
 *    default stream.  Calls are stream-ordered and keep no global mutable
 *    state besides a per-process cache of kernel attributes.
 *  - Return value: PRRP_OK or one of the status codes below; the error
 *    record carries the payload the reference attaches to its exceptions.
 */
#ifndef PRRP_B200_H
#define PRRP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; each maps onto the reference's exception contract
 * (errors.py:4-54, luprrp.py:143-150). */
enum prrp_status {
  PRRP_OK = 0,
  PRRP_ERR_DIM = 1,              /* DimensionMismatch (errors.py:4-5)              */
  PRRP_ERR_ARG = 2,              /* ValueError: b out of range, tau <= 1, ...       */
  PRRP_ERR_RANK_DEFICIENT = 3,   /* RankDeficient(index)   (errors.py:30-38)        */
  PRRP_ERR_NONCONVERGENCE = 4,   /* NonConvergence(worst)  (errors.py:41-50)        */
  PRRP_ERR_SINGULAR_MATRIX = 5,  /* SingularMatrix(column) (errors.py:19-27)        */
  PRRP_ERR_SINGULAR_FACTOR = 6,  /* SingularFactor(index)  (errors.py:8-16)         */
  PRRP_ERR_CUDA = 7,             /* CUDA runtime failure (message in err->msg)      */
  PRRP_ERR_UNSUPPORTED = 8,      /* shape outside the device path (e.g. b > 128)    */
  PRRP_ERR_NCCL = 9
};

/* Error payload: the attributes the reference sets on its exceptions
 * (exc.index / exc.column / exc.worst, exc.panel at luprrp.py:172-174,192-194,
 * exc.tree_node at tournament.py:182-184). */
typedef struct prrp_err {
  int32_t code;        /* prrp_status                                       */
  int32_t panel;       /* panel index, -1 if not attached                   */
  int32_t index;       /* RankDeficient / SingularFactor index, else -1     */
  int32_t column;      /* SingularMatrix column, else -1                    */
  int32_t tree_level;  /* CALU tournament node, -1 if none                  */
  int32_t tree_index;
  double worst;        /* NonConvergence: largest multiplier still > tau    */
  char msg[160];
} prrp_err;

/* ElimStats scalars (luprrp.py:33-78).  Flop counters are exact rationals in
 * the reference; the shim rebuilds them on the host from swap_counts. */
typedef struct prrp_stats {
  double original_max;
  double intermediate_max;
  double finish_max;
  double panel_multiplier_max;
  int64_t total_swaps;
} prrp_stats;

/* Optional device-time breakdown of a factorization (CUDA events around
 * every launch, summed per kernel class).  Classes: */
enum prrp_kclass {
  PRRP_K_PANEL = 0,      /* panel_qrcp_kernel    (cluster QRCP)            */
  PRRP_K_TRSM = 1,       /* trsm_kernel          (L21, tau candidates)     */
  PRRP_K_FINALIZE = 2,   /* panel_finalize_kernel (swap loop, GEPP A11)    */
  PRRP_K_PERMUTE = 3,    /* permute_kernel                                 */
  PRRP_K_SCHUR = 4,      /* schur_dmma_kernel / schur_simt_kernel          */
  PRRP_K_COMPOSE = 5,    /* compose_kernel                                 */
  PRRP_K_BLOCKROW = 6,   /* blockrow kernels (GEPP finish of the block row) */
  PRRP_K_GEPP = 7,       /* gepp_diag_kernel (b x b diagonal block GEPP)   */
  PRRP_K_OTHER = 8,      /* init kernels                                   */
  PRRP_K_COUNT = 9
};

typedef struct prrp_timing {
  double ms[PRRP_K_COUNT];       /* summed event time per class             */
  int32_t launches[PRRP_K_COUNT];
  double schur_flops;            /* algorithmic 2*M*N*K summed over updates */
  double total_ms;               /* first to last event of the call         */
} prrp_timing;

/* Library identification: returns the ABI version (major*100 + minor). */
int prrp_b200_abi_version(void);

/* Probe the device: writes SM count and whether 16-CTA clusters are
 * available; returns PRRP_OK or PRRP_ERR_CUDA. */
int prrp_b200_device_probe(int32_t* sm_count, int32_t* max_cluster, prrp_err* err);

/* LU_PRRP factorization, Algorithm 1 — replaces prrp.luprrp_factor
 * (luprrp.py:153-201).  A: m x n row-major device matrix (m >= n), factored
 * in place into packed L\U.  perm: device int64[m].  swap_counts: host
 * int32[ceil(n/b)] (ElimStats.swap_counts).  Requires 1 <= b <= min(n,128)
 * for the device panel engine (b > 128 returns PRRP_ERR_UNSUPPORTED). */
int prrp_luprrp(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau,
                int64_t* perm, int32_t* swap_counts, prrp_stats* stats, prrp_err* err,
                void* stream);

/* prrp_luprrp with an optional per-kernel-class device-time breakdown
 * (timing may be NULL; then identical to prrp_luprrp). */
int prrp_luprrp_timed(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau,
                      int64_t* perm, int32_t* swap_counts, prrp_stats* stats, prrp_err* err,
                      prrp_timing* timing, void* stream);

/* Sustained FP64 tensor-pipe (DMMA.8x8x4) throughput of this device in
 * TFLOP/s: register-resident mma.sync.m8n8k4.f64 loop on every SM for about
 * `ms` milliseconds.  The roofline denominator of the Schur update. */
int prrp_b200_dmma_peak(double ms, double* tflops, prrp_err* err);

/* CALU_PRRP factorization with a binary tournament tree of `leaf_count`
 * leaves — replaces prrp.caluprrp_factor(a, b, tau, binary_tree(P))
 * (tournament.py:237-296); leaf_count == 0 selects flat_tree()
 * (tournament.py:81-88, 202-208).  Arguments as prrp_luprrp, plus
 * tournament_charge3 (host int64[ceil(n/b)], may be NULL): 3x the
 * tournament flop charge of each panel (tournament.py:224-234), -1 for a
 * single-node panel, so the caller can rebuild the exact rational counters. */
int prrp_caluprrp(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau,
                  int32_t leaf_count, int64_t* perm, int32_t* swap_counts, int64_t* tournament_charge3,
                  prrp_stats* stats, prrp_err* err, void* stream);

/* Kernel launches in the CUDA graph the calling thread's last prrp_caluprrp
 * replayed (diagnostics / the bench's launch count; 0 before any call). */
int64_t prrp_b200_graph_kernels(void);

/* Diagnostics: average device time (ms) of the panel QRCP engine alone
 * (qr_column_pivoting, pivoted_qr.py:74-87) on an h x p transposed panel
 * whose columns are the rows of `a` (device, row-major, lda), `reps`
 * launches between CUDA events.  nwc / cpt > 0 force a latency-engine shape
 * (compute warps per CTA, columns per 8-thread team), 0 = the default
 * choice; nwc < 0 runs the thread-per-column engines (h = 64 or 128).
 * ctas_out = cluster size used.  R_out (device, column-major h x p: R by
 * position) and perm_out (device, p column indices) optionally return the
 * last launch's result (both or neither), so every engine shape can be
 * checked against the oracle. */
int prrp_b200_qrcp_time(const double* a, int64_t lda, int32_t h, int64_t p, int32_t nwc, int32_t cpt, int32_t reps,
                        double* ms_out, int32_t* ctas_out, double* R_out, int64_t* perm_out, prrp_err* err);

/* prrp_caluprrp through the direct (uncaptured) enqueue with every launch
 * timed by CUDA events on its stream (per kernel class, as
 * prrp_luprrp_timed); timing may be NULL. */
int prrp_caluprrp_timed(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, double tau,
                        int32_t leaf_count, int64_t* perm, int32_t* swap_counts, int64_t* tournament_charge3,
                        prrp_stats* stats, prrp_err* err, prrp_timing* timing, void* stream);

/* Tournament-pivoted GEPP ("calu_factor") with a binary tree of
 * `leaf_count` leaves, 0 = flat tree — replaces prrp.calu_factor(a, b, tree)
 * (tournament.py:299-359): every tournament node selects by partial
 * pivoting (tournament.py:142-150), the block row is finished by GEPP
 * without composing L21, L21 = A21 U11^-1 (matcore.py:97-113).  Arguments
 * as prrp_caluprrp without tau and swap counts (always 0 for this
 * factorization); tournament_charge3[k] = 3x panel k's tournament flop
 * charge (tournament.py:220-234), 0 when the panel has no selection. */
int prrp_calu(double* A, int64_t lda, int64_t m, int64_t n, int32_t b, int32_t leaf_count,
              int64_t* perm, int64_t* tournament_charge3, prrp_stats* stats, prrp_err* err,
              void* stream);

/* One GEPP selector node (tournament.py:142-150): partial pivoting on the
 * r x cols row-major device matrix `a` (r > cols, cols <= 128); order
 * (device int64[r]) = the elimination's row order, *count (host) = rows
 * chosen before the first zero pivot (cols when none). */
int prrp_gepp_select(const double* a, int64_t lda, int64_t r, int32_t cols, int64_t* order,
                     int32_t* count, prrp_err* err, void* stream);

/* gepp_factor of an m x n row-major device matrix of any shape (gepp.py:39-65),
 * in place: packed L\U (unit lower multipliers below the diagonal), row
 * order perm (device int64[m]), running max of the live trailing block
 * (intermediate_max) and max|A| (original_max), host doubles.  A zero pivot
 * column k -> PRRP_ERR_SINGULAR_MATRIX with err->column = k. */
int prrp_gepp(double* A, int64_t lda, int64_t m, int64_t n, int64_t* perm, double* intermediate_max,
              double* original_max, prrp_err* err, void* stream);

/* Strong RRQR of an h x p matrix `a` (column-major, lda >= h) with leading
 * block size bsel <= h and threshold tau — replaces prrp.strong_rrqr
 * (pivoted_qr.py:113-147).  Outputs (device, column-major): R h x p (ldr=h),
 * Q h x h, perm int64[p], Lblk (p-bsel) x bsel.  swap_count: host int32.
 * Requires h <= 128, p >= bsel+1, h >= bsel. */
int prrp_strong_rrqr(const double* a, int64_t lda, int32_t h, int64_t p, int32_t bsel,
                     double tau, double* R, double* Q, int64_t* perm, double* Lblk,
                     int32_t* swap_count, prrp_err* err, void* stream);

/* Unpivoted Householder QR of an h x p column-major matrix — replaces
 * prrp.householder_qr (pivoted_qr.py:64-71).  R h x p, Q h x h (device). */
int prrp_householder_qr(const double* a, int64_t lda, int32_t h, int64_t p,
                        double* R, double* Q, prrp_err* err, void* stream);

/* Multiplier block (R11^-1 R12)^T of an upper-trapezoidal R (column-major,
 * ldr >= b, p columns) — replaces prrp.multiplier_block (pivoted_qr.py:90-98):
 * back substitution with true division, SingularFactor on an exact zero
 * diagonal.  L: (p-b) x b column-major (ldl >= p-b), device.  absmax (host,
 * may be NULL) receives max|L|. */
int prrp_multiplier_block(const double* R, int64_t ldr, int32_t b, int64_t p, double* L, int64_t ldl,
                          double* absmax, prrp_err* err, void* stream);

/* Rank-K Schur update C <- C - L*B with the reference's rounding recipe
 * (matcore.rank_update, matcore.py:54-61: product accumulated in increasing
 * k from zero, then one subtraction).  C: M x N row-major (ldc), L: M x K
 * column-major (ldl), B: K x N row-major (ldb).  absmax (host, may be NULL)
 * receives max|C_new|.  K must be a multiple of 4, <= 128. */
int prrp_schur_update(double* C, int64_t ldc, const double* L, int64_t ldl,
                      const double* B, int64_t ldb, int64_t M, int64_t N, int32_t K,
                      double* absmax, prrp_err* err, void* stream);

/* Partial-pivoting LU of an m x n row-major device matrix in place —
 * replaces prrp.gepp_factor (gepp.py:39-65) for the b x w block-row shapes
 * the factorizations use (m <= 128).  perm: device int64[m];
 * intermediate_max: host double. */
int prrp_gepp_blockrow(double* A, int64_t lda, int32_t m, int64_t n, int64_t* perm,
                       double* intermediate_max, prrp_err* err, void* stream);

/* QR with column pivoting over min(h, p) steps of an h x p column-major
 * matrix — replaces prrp.qr_column_pivoting (pivoted_qr.py:74-87): exact
 * numpy-pairwise column norms each step, first maximum, Householder steps
 * of _reflect.  R h x p, Q h x h (column-major), perm int64[p] (device).
 * Requires h <= 128. */
int prrp_qrcp(const double* a, int64_t lda, int32_t h, int64_t p, double* R, double* Q,
              int64_t* perm, prrp_err* err, void* stream);

/* Verification: resid_sq = ||Pi A - L U||_F^2 and
 * a_sq = ||A||_F^2 (host doubles) for packed factors LU (m x n row-major,
 * unit lower L below the diagonal, U on and above) of the m x n row-major A
 * with row order perm (device int64[m]) — the quantities of
 * prrp.metrics.rel_factorization_error (metrics.py:56-63). */
int prrp_lu_residual(const double* A, int64_t lda, const double* LU, int64_t ldlu,
                     const int64_t* perm, int64_t m, int64_t n, double* resid_sq, double* a_sq,
                     prrp_err* err, void* stream);

/* Solve A X = B with the packed square factors — replaces prrp.luprrp_solve
 * (luprrp.py:204-214).  B, X: n x nrhs column-major (device); SingularFactor
 * on an exact-zero U diagonal. */
int prrp_lu_solve(const double* LU, int64_t ldlu, int64_t n, const int64_t* perm, const double* B,
                  int64_t ldb, double* X, int64_t ldx, int32_t nrhs, prrp_err* err, void* stream);

/* ---- Distributed CALU_PRRP, one process per GPU (
 * PAPER.md:1739-1751 layout, 2885-2951 per-panel pattern).  Replaces
 * prrp.caluprrp_factor (tournament.py:237-296) when the matrix is spread
 * over `nranks` GPUs: column block-cyclic (process grid 1 x nranks, block b):
 * global column block J lives on rank J mod nranks as local block
 * J div nranks, all m rows (A_loc row-major m x n_loc, lda even).  The
 * library does not communicate: per panel k the caller runs
 *     owner (k mod nranks):  prrp_calu_dist_select(k)
 *     everyone:              broadcast msg[k & 1][0 .. msg_bytes(k)) from the owner
 *                            prrp_calu_dist_apply(k, 0)
 * (the owner of panel k+1 may run apply(k, 1), select(k+1), apply(k, 2):
 * look-ahead), then prrp_calu_dist_stats, a MAX all-reduce of the int64
 * stats record over the ranks, and prrp_calu_dist_finish.  Every rank ends
 * with the same perm (device, m) and its columns of the packed L\U; the
 * results are bit-identical to prrp_caluprrp on one GPU. */
int prrp_calu_dist_create(void** handle, double* A_loc, int64_t lda, int64_t m, int64_t n, int64_t n_loc,
                          int32_t b, double tau, int32_t leaf_count, int32_t nranks, int32_t rank,
                          int64_t* perm, prrp_err* err, void* stream);
/* Device buffers: the two panel messages (parity k & 1), their capacity in
 * bytes, and the int64 statistics record to be MAX-reduced (length). */
int prrp_calu_dist_buffers(void* handle, void** msg0, void** msg1, int64_t* msg_capacity, void** stats,
                           int64_t* stats_len);
/* Bytes of panel k's message that must be broadcast (-1 on a bad panel). */
int64_t prrp_calu_dist_msg_bytes(void* handle, int32_t panel);
int prrp_calu_dist_select(void* handle, int32_t panel, prrp_err* err, void* stream);
/* part: 0 = all, 1 = head (all but the trailing update beyond the next
 * panel's block), 2 = tail (that update). */
int prrp_calu_dist_apply(void* handle, int32_t panel, int32_t part, prrp_err* err, void* stream);
int prrp_calu_dist_stats(void* handle, prrp_err* err, void* stream);
/* reduced: the MAX-reduced statistics record (device; NULL = this rank's own).
 * Outputs as prrp_caluprrp; the error is the owner's first failure (every
 * rank reports the same). */
int prrp_calu_dist_finish(void* handle, const int64_t* reduced, int32_t* swap_counts,
                          int64_t* tournament_charge3, prrp_stats* stats, prrp_err* err, void* stream);
void prrp_calu_dist_destroy(void* handle);

/* ---- Stability measurements (metrics.py:65-145) on device buffers.
 * r = rhs - A x with the reference's compensated accumulation
 * (residual_extended, metrics.py:75-92: Veltkamp two-product + Knuth
 * two-sum per term, j ascending): bit-identical to the reference.  A is
 * row-major m x n; x (n), rhs and r (m) are device vectors. */
int prrp_residual_extended(const double* A, int64_t lda, int64_t m, int64_t n, const double* x,
                           const double* rhs, double* r, prrp_err* err, void* stream);
/* Absolute sums: colabs[j] = sum_i |A_ij| (||A||_1 = max), rowabs[i] =
 * sum_j |A_ij| (||A||_inf), absax[i] = sum_j |A_ij| |x_j| (the componentwise
 * denominator |A| |x|, metrics.py:109); any output may be NULL.  Summation
 * order: per column / per warp (the reference uses numpy / BLAS orders). */
int prrp_abs_sums(const double* A, int64_t lda, int64_t m, int64_t n, const double* x, double* colabs,
                  double* rowabs, double* absax, prrp_err* err, void* stream);

/* prrp_gepp whose running maximum covers only the entries each step
 * updates (max over steps k of max|A[k+1:, k+1:]| after step k): the
 * block variants' finish statistic (block_variants.py:170-186). */
int prrp_gepp_steps(double* A, int64_t lda, int64_t m, int64_t n, int64_t* perm, double* steps_max,
                    double* original_max, prrp_err* err, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PRRP_B200_H */
