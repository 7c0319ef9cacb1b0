/*
 * tsvd.h - C ABI of the B200-native truncated SVD hot path.
 *
 * Implements the block iteration shared by RandSVD (Alg. 1)
 * and LancSVD (Alg. 2) of Tomas, Quintana-Orti, Anzt,
 * "Fast Truncated SVD of Sparse and Dense Matrices on Graphics Processors"
 * (arXiv 2403.06218).  Citations "P:<line>" refer to PAPER.md.
 *
 * Problem (Sec. 2): A in R^{m x n}, m >= n, given as CSR or
 * dense; compute U_r (m x r), Sigma_r = diag(sigma_1..sigma_r) descending,
 * V_r (n x r) with A ~ U_r Sigma_r V_r^T (Eq. 2).
 *
 * Conventions
 *  - FP64 only (IEEE binary64).  Integers: int64 row pointers, int32
 *    column indices (n < 2^31).
 *  - Every dense block crossing this ABI is ROW-MAJOR with an explicit
 *    leading dimension (elements).  U is m x r (ldu >= r), V is n x r.
 *  - mem_kind: TSVD_HOST (pageable or pinned host memory) or TSVD_DEVICE
 *    (device memory on the current CUDA device).
 *  - Ownership: create* COPIES A into library-owned device memory; the caller
 *    keeps its buffers.  get copies into caller buffers.  destroy frees all.
 *  - Errors: every call returns a tsvd_status; nothing is thrown, nothing
 *    aborts.  After a negative status the handle stays valid for destroy.
 *    Non-convergence is the positive warning TSVD_WARN_NOTCONV (results of
 *    the last cycle are retrievable).  A Cholesky breakdown is not an error:
 *    the CGS2 fallback of P:275 handles it.
 *  - Threading: a handle is not thread-safe; distinct handles may run
 *    concurrently on distinct streams.  All work is ordered on the handle's
 *    stream (tsvd_set_stream); calls return after the stream work they
 *    enqueue has completed unless documented otherwise.
 *  - There is no CPU fallback: if no CUDA device is usable every entry point
 *    that needs one returns TSVD_ECUDA.
 */
#ifndef TSVD_H
#define TSVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsvd_ctx* tsvd_t;
typedef int tsvd_status;

enum {
  TSVD_OK = 0,
  TSVD_WARN_NOTCONV = 1, /* maxit reached before max_{i<=r} rho_i <= tol*sigma_1 */
  TSVD_WARN_FALLBACK = 2, /* tsvd_dbg_cholqr2 / _cgs_cqr2 only: the Cholesky breakdown
                             test fired and the CGS2 fallback gave the result */
  TSVD_WARN_SVD = 3,     /* the device Jacobi SVD of B_k / R_p (reading R20) hit its
                            sweep cap (60) before every column pair passed the
                            rotation test; results retrievable, tsvd_info counts it */
  TSVD_EINVAL = -1,      /* bad argument (NULL, non-canonical CSR, tol <= 0 ...) */
  TSVD_ESHAPE = -2,      /* m < n, r > n, d % b != 0, r > d, r + p > n ...     */
  TSVD_ENOMEM = -3,      /* device allocation failed                            */
  TSVD_ECUDA = -4,       /* CUDA runtime error / no usable device               */
  TSVD_ENCCL = -5,       /* NCCL missing or failed (multi-GPU handles)          */
  TSVD_ESTATE = -6       /* e.g. tsvd_get before a successful solve             */
};

enum { TSVD_HOST = 0, TSVD_DEVICE = 1 };
enum { TSVD_ROW_MAJOR = 0, TSVD_COL_MAJOR = 1 };

/* ---- creation ----------------------------------------------------------
 * tsvd_create_csr: A as CSR.  rowptr[m+1] (rowptr[0] = 0,
 * non-decreasing, rowptr[m] = nnz), colidx[nnz] in [0, n), vals[nnz].  The
 * columns of a row may be unsorted and may repeat: the library's copy is
 * canonicalised on the device (columns sorted within each row, duplicate
 * entries summed in their input order).  The library builds
 * CSR(A^T) on the device (radix sort by column, stable) so that A^T.X needs
 * no atomics (north_star; P:460 discusses the transposed product).
 * Returns TSVD_ESHAPE if m < n ("otherwise target the transpose"),
 * TSVD_EINVAL if the row pointer is malformed or a column index is out of
 * range. */
tsvd_status tsvd_create_csr(tsvd_t* h, int64_t m, int64_t n, int64_t nnz,
                            const int64_t* rowptr, const int32_t* colidx,
                            const double* vals, int mem_kind);

/* tsvd_create_dense: dense A (Table 1 caption P:327: the products become
 * GEMMs).  layout TSVD_ROW_MAJOR (lda >= n) or TSVD_COL_MAJOR (lda >= m);
 * stored row-major on the device. */
tsvd_status tsvd_create_dense(tsvd_t* h, int64_t m, int64_t n, const double* A,
                              int64_t lda, int layout, int mem_kind);

/* ---- multi-GPU (row-partitioned) creation, SURVEY 8(e) ---------------------
 * One process per GPU.  Rank g owns rows [row_begin, row_end) of A (the
 * caller chooses them, e.g. balanced by nnz: tsvd_partition_rows) and the
 * n-shard [g*ns, min(n, (g+1)*ns)) of every n-side vector, ns = ceil(n/world).
 * The ranks share a 128-byte ncclUniqueId created by one of them with
 * tsvd_nccl_unique_id and broadcast by the harness (torch.distributed).
 * Per Lanczos block step the ranks exchange: a reduce-scatter of A_g^T Qbar_i,
 * an all-gather of Q_i, and all-reduces of the b x b / s x b projections and
 * Gram matrices; B_k, its SVD, rho and the restart are replicated.
 * tsvd_get then returns this rank's rows of U (row_end-row_begin) and its
 * n-shard of V.  All ranks must call every solver entry point collectively. */
typedef struct {
  int rank, world;
  const void* nccl_id;        /* 128 bytes, identical on all ranks */
  int64_t m_global, n_global; /* sizes of the whole A, m >= n */
  int64_t row_begin, row_end; /* this rank's rows of A */
  void* loopback;             /* NULL (NCCL), or a tsvd_loopback_create group:
                                 then nccl_id may be NULL (test-only, below) */
} tsvd_dist;
/* rowptr/colidx/vals: this rank's rows only (local rowptr starting at 0,
 * GLOBAL column indices). */
tsvd_status tsvd_create_csr_dist(tsvd_t* h, const tsvd_dist* dist, int64_t nnz_local,
                                 const int64_t* rowptr, const int32_t* colidx,
                                 const double* vals, int mem_kind);
/* A: this rank's (row_end - row_begin) x n_global rows, row-major, lda >= n. */
tsvd_status tsvd_create_dense_dist(tsvd_t* h, const tsvd_dist* dist, const double* A,
                                   int64_t lda, int mem_kind);
/* Fill out128 with a fresh ncclUniqueId (TSVD_ENCCL if NCCL is unavailable). */
tsvd_status tsvd_nccl_unique_id(void* out128);
/* TEST-ONLY in-process communicator: `world` (1..8) handles on ONE device,
 * each driven from its own host thread, exchange through device memory
 * instead of NCCL (rank-ordered sums), so the library's complete
 * row-partitioned code path runs at world > 1 on a single GPU.  Pass the
 * group as tsvd_dist.loopback to every rank's create call; destroy it after
 * all its handles.  Collectives block the calling thread until all ranks
 * reach them (like NCCL's), so the ranks MUST run on separate threads. */
tsvd_status tsvd_loopback_create(int world, void** group);
tsvd_status tsvd_loopback_destroy(void* group);
/* Row split of a CSR row pointer (host) into `world` contiguous ranges with
 * (nearly) equal nonzeros: bounds[0] = 0 ... bounds[world] = m. */
tsvd_status tsvd_partition_rows(const int64_t* rowptr, int64_t m, int world, int64_t* bounds);

/* ---- options ----------------------------------------------------------- */
/* cudaStream_t to order all work on (e.g. torch.cuda.current_stream()).
 * NULL => the legacy default stream.  Until this is called a handle uses a
 * library-owned non-blocking stream. */
tsvd_status tsvd_set_stream(tsvd_t h, void* cuda_stream);
/* Philox4x32-10 seed for the start block (draw 0) and for breakdown
 * replacement columns (draws 1, 2, ...).  P:406, reading R9. */
tsvd_status tsvd_set_seed(tsvd_t h, uint64_t seed);
/* Krylov dimension d of LancSVD (the paper's "r"); must be a
 * multiple of b with r <= d <= n and d <= 1536 (the largest B_k the device
 * Jacobi SVD takes; checked when the solve starts: TSVD_ESHAPE).  0 =>
 * default min(n, max(4r, 2b), 1536) rounded down to a multiple of b. */
tsvd_status tsvd_set_krylov_dim(tsvd_t h, int d);
/* Restart of LancSVD.  keep = 0 (default): the paper's restart, Alg. 2 S7
 * (P:200-203): the next cycle starts from the first b left Ritz vectors.
 * keep = l > 0: THICK restart (SURVEY 8(f) N1 -- the paper's future work,
 * P:212/P:500, after Baglama-Reichel, ref. [2] P:509): the l largest Ritz
 * pairs are kept as the first l columns of the next cycle's bases, Qbar_{k+1}
 * follows them, and the block recurrence continues for (d - l)/b steps; the
 * projected matrix becomes [Sigma_l 0; S L_1 ...] with S = Rbar_k Vbar[last
 * b rows, :l] (derivation: oracle/lancsvd.py header).  Requirements checked
 * at solve time: l % b == 0 and r <= l < d, else TSVD_ESHAPE.  keep < 0 =>
 * TSVD_EINVAL. */
tsvd_status tsvd_set_thick_restart(tsvd_t h, int keep);
/* Device memory: every library allocation (A, CSR(A^T), bases, workspaces)
 * is stream-ordered (cudaMallocAsync on the handle's stream) from the current
 * device's default memory pool; at first use the pool's release threshold is
 * raised so blocks freed by tsvd_destroy stay reserved for the next handle
 * (no cudaMalloc per solve).  tsvd_trim_memory synchronises the device and
 * returns reserved-but-unused pool memory above keep_bytes to the system.
 * Returns TSVD_ECUDA without a usable device. */
tsvd_status tsvd_trim_memory(size_t keep_bytes);
/* Device memory from the caller instead (e.g. PyTorch's caching
 * allocator).  Process-wide: every later library allocation (create, solver
 * workspaces) calls alloc(bytes, stream, ctx) with the handle's cudaStream_t
 * and must get device memory usable in stream order on that stream, or NULL
 * (=> TSVD_ENOMEM); such blocks are returned with free_(ptr, stream, ctx)
 * (stream-ordered: work already enqueued on `stream` may still use the block
 * until it completes).  Blocks obtained before a change go back to the
 * allocator that produced them.  alloc = NULL restores the default pool.
 * Both callbacks must be thread-safe if handles are used from several threads;
 * they are never called with a lock of the library held. */
typedef void* (*tsvd_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*tsvd_free_fn)(void* ptr, void* stream, void* ctx);
tsvd_status tsvd_set_allocator(tsvd_alloc_fn alloc, tsvd_free_fn free_, void* ctx);
/* Where the outputs U_r = Pbar_k Ubar[:, :r], V_r = P_k Vbar[:, :r] (Eq. 12;
 * RandSVD Alg. 1 S6/S7) are formed.  TSVD_OUT_AUTO (default): in separate
 * result buffers when (m + n) r doubles fit in the free device memory, else
 * in place.  TSVD_OUT_SEPARATE: always separate buffers.  TSVD_OUT_INPLACE:
 * over the first r columns of the bases themselves (row-local products,
 * computed in row chunks through the pass scratch buffer, so no m x r buffer
 * is allocated: what lets C5 -- m = n = 5e7, d = 160, 141 GB of bases -- run
 * on one 180 GB GPU).  The bases are then overwritten; results are read by
 * tsvd_get as usual.  Other values => TSVD_EINVAL. */
enum { TSVD_OUT_AUTO = 0, TSVD_OUT_SEPARATE = 1, TSVD_OUT_INPLACE = 2 };
tsvd_status tsvd_set_output_mode(tsvd_t h, int mode);
/* Block orthogonalisation of every S3b / S5 step (and of RandSVD's CGS-QR
 * panels).  TSVD_ORTHO_CGS_CQR2 (default): the paper's Alg. 5.
 * TSVD_ORTHO_BCGS_PIP2: BCGS-PIP+ (reading R34 --
 * not in the paper): two Pythagorean block-CGS passes, each needing ONE
 * reduction [P Y]^T Y (multi-GPU: 2 all-reduces per orthogonalisation
 * instead of 4) and no basis-free TRSM / Gram passes; the same Cholesky
 * breakdown test and CGS2 fallback.  Stable while the block is not
 * nearly inside span(P) (kappa(Y) well below u^{-1/2}); a measured ablation.
 * Other values => TSVD_EINVAL. */
enum { TSVD_ORTHO_CGS_CQR2 = 0, TSVD_ORTHO_BCGS_PIP2 = 1 };
tsvd_status tsvd_set_ortho(tsvd_t h, int ortho);
/* CUDA-graph replay of a LancSVD cycle's block steps (single-GPU handles):
 * with on != 0 the deferred-check pass of a cycle (no host synchronisation
 * inside) is captured the second time the same cycle shape runs and replayed
 * afterwards; results are bit-identical to the eager path.  Default off (no
 * measured gain on C2); env TSVD_GRAPHS=1 sets it for new
 * handles. */
tsvd_status tsvd_set_graphs(tsvd_t h, int on);
/* Panel width of CGS-QR (Alg. 3) inside RandSVD; default 16. */
tsvd_status tsvd_set_qr_block(tsvd_t h, int b_qr);
/* Optional exact start block instead of the Philox one: for LancSVD the
 * m x b block G that S1 orthonormalises; for RandSVD the n x l block Q_0.
 * Row-major, leading dimension ld.  The block is copied; it is used by every
 * later solve on this handle until tsvd_set_start(h, NULL, 0, 0). */
tsvd_status tsvd_set_start(tsvd_t h, const double* block, int64_t rows,
                           int64_t cols, int64_t ld, int mem_kind);

/* ---- solvers ------------------------------------------------------------
 * tsvd_block_lanczos: Alg. 2 with both-side full reorthogonalisation
 * (CGS-CQR2, Alg. 5) and the basic restart of [9], restart block
 * re-orthonormalised (reading R11).  Cycles until
 * max_{i<=r} ||Rbar_k Vbar[last b rows, i]||_2 <= tol * sigma_1 (from Eq. 10,
 * reading R12) or maxit cycles.  r >= 1 wanted triplets, b >= 1 block size
 * (any width: blocks wider than 32 are orthogonalised in 32-column panels as
 * Alg. 3 does), tol > 0, maxit >= 1. */
tsvd_status tsvd_block_lanczos(tsvd_t h, int r, int b, double tol, int maxit);
/* tsvd_block_lanczos_threshold (Eq. 3): the rank r
 * is set by the threshold ||A - U_r S_r V_r^T||_2 = sigma_{r+1} <= tau *
 * sigma_1.  Reading R33: tsvd_block_lanczos is run for r + 1
 * wanted triplets (r = b first, then doubled up to r_max, each solve from a
 * fresh start with the handle's Krylov dimension or the default for r + 1);
 * the result is the smallest r whose sigma_{r+1} <= tau * sigma_1 with
 * triplets 1..r+1 converged (rho <= tol).  *r_out (may be NULL) receives r;
 * tsvd_get then returns r columns.  0 < tau < 1, b >= 1, r_max >= 1 (capped
 * at n - 1), else TSVD_EINVAL.  Not found by r_max: TSVD_WARN_NOTCONV with
 * r = r_max triplets retrievable. */
tsvd_status tsvd_block_lanczos_threshold(tsvd_t h, double tau, int b, double tol, int maxit,
                                         int r_max, int* r_out);
/* tsvd_rsvd: Alg. 1 with l = r + p columns (p = oversampling) and q power
 * iterations, i.e. q + 1 passes of S1-S4 (paper p = q + 1, reading R6); QR by
 * CGS-QR (Alg. 3) with panels of b_qr columns.  l <= min(n, 1536) (the
 * l x l R_p goes through the device Jacobi SVD), else TSVD_ESHAPE before any
 * work is done. */
tsvd_status tsvd_rsvd(tsvd_t h, int r, int p, int q);

/* ---- results ------------------------------------------------------------
 * Copies U_r (m x r, row-major, ldu >= r), S (r), V_r (n x r, ldv >= r) of
 * the last solve.  Any pointer may be NULL to skip it.  Sign convention: the
 * largest-|.| entry of each v_i is positive (lowest index on ties). */
tsvd_status tsvd_get(tsvd_t h, double* U, int64_t ldu, double* S, double* V,
                     int64_t ldv, int mem_kind);

/* Explicit residuals of the last solve's r triplets (Eq. 14,
 * P:408-410, as corrected by DESIGN.md reading R13: the printed
 * ||A u_i - sigma_i v_i|| is dimensionally inconsistent):
 *   e[i] = ||A v_i - sigma_i u_i||_2 / sigma_1   (north_star's measure)
 *   rel[i] = ||A v_i - sigma_i u_i||_2 / sigma_i (the paper's R_i)
 * computed on the device with the library's own A.X product and a
 * fixed-order column-norm reduction (multi-GPU: row-sharded sums
 * all-reduced; every rank gets all r values).  e, rel: host arrays of r
 * doubles, either may be NULL.  Collective on multi-GPU handles.
 * TSVD_ESTATE before a successful solve. */
tsvd_status tsvd_residuals(tsvd_t h, double* e, double* rel);

typedef struct {
  int cycles;       /* LancSVD restart cycles run (RandSVD: q + 1)        */
  int nconv;        /* i < r with rho_i <= tol*sigma_1 (LancSVD)          */
  int r, d, b;      /* parameters of the last solve (RandSVD: d = l)      */
  int breakdowns;   /* orthogonalisations whose Cholesky breakdown test
                       fired and that the CGS2 fallback redid     */
  double rho_max;   /* max_{i<r} rho_i / sigma_1 (LancSVD)                */
  double sigma1;
  double ms_total;  /* device time of the last solve (CUDA events)        */
  int64_t launches; /* kernels launched by the last solve                 */
  int replaced;     /* dependent columns the fallback replaced by Philox
                       draws (reading R16)                                */
  int svd_sweeps;   /* largest Jacobi sweep count of the solve's SVDs     */
  int svd_unconverged; /* SVDs that hit the sweep cap (=> TSVD_WARN_SVD)  */
} tsvd_info;
tsvd_status tsvd_get_info(tsvd_t h, tsvd_info* out);
/* rho_i / sigma_1 for i < r of the last LancSVD cycle (host buffer). */
tsvd_status tsvd_get_rho(tsvd_t h, double* rho);

/* Per-phase device-time instrumentation (CUDA events on the handle's stream
 * around each phase call).  Phases (index: name): 0 apply_A (A.X, Alg. 2
 * S4 / Alg. 1 S1), 1 apply_AT (A^T.X, S2 / S3), 2 ortho_tn (gemm_tn passes
 * of Alg. 4/5), 3 ortho_nn (gemm_nn passes of Alg. 4/5 against the basis),
 * 4 ortho_small (b x b Cholesky / reductions), 5 small_svd, 6 restart_out
 * (restart product, outputs, sign), 7 other, 8 ortho_rowT (the basis-free
 * passes: Gram of Y and the TRSM-as-multiply S L^{-T}), 9 beside_svd (the
 * last block step's m-side product and orthogonalisation when they run
 * beside the Jacobi SVD of B_k on the SMs it leaves free -- kept apart so
 * the other phases measure kernels that have the GPU to themselves).
 * bytes/flops are
 * ALGORITHMIC (compulsory) counts per DESIGN.md "Roofline", not measured
 * traffic.  Aggregates accumulate over solves until reset. */
typedef struct {
  const char* name;   /* static string */
  int64_t calls;      /* phase calls */
  int64_t launches;   /* kernels launched inside them */
  double ms;          /* summed event time */
  double bytes;       /* summed algorithmic bytes */
  double flops;       /* summed algorithmic flops */
} tsvd_prof_entry;
enum { TSVD_NPROF = 10 };
tsvd_status tsvd_set_profiling(tsvd_t h, int on);
/* Record only the phases whose bit (1 << phase index above) is set in
 * `mask` (0 = off; tsvd_set_profiling(h, 1) = all phases).  Each recorded
 * phase call adds two event records to the stream; bench.py times its
 * solves with only the dominant phase recorded (the roofline needs that
 * phase's event time) and takes the full breakdown from a separate solve. */
tsvd_status tsvd_set_profiling_mask(tsvd_t h, unsigned mask);
tsvd_status tsvd_get_profile(tsvd_t h, tsvd_prof_entry* out /* TSVD_NPROF */);
tsvd_status tsvd_reset_profile(tsvd_t h);

tsvd_status tsvd_destroy(tsvd_t h);
const char* tsvd_strerror(tsvd_status s);
/* Message of the last failing call on this thread ("" if none). */
const char* tsvd_last_error(void);

/* ---- single-kernel entry points for parity tests (same library) ---------
 * All pointers are DEVICE pointers, row-major with the given leading
 * dimensions, work is enqueued on `stream` (NULL = legacy default) and the
 * call synchronises that stream before returning. */

/* Philox normal block (reading R9): out[i*ld + j] = G(row0+i, j) of a
 * q_total x w block, seed, draw. */
tsvd_status tsvd_dbg_philox(double* out, int64_t q, int w, int64_t ld,
                            uint64_t seed, uint64_t draw, int64_t row0,
                            int64_t q_total, void* stream);
/* Raw Philox4x32-10 words for (ctr, key) pairs: ctr[4*i..], key[2*i..] ->
 * out[4*i..] (uint32).  count pairs.  Pointers are device pointers. */
tsvd_status tsvd_dbg_philox_words(const uint32_t* ctr, const uint32_t* key,
                                  uint32_t* out, int64_t count, void* stream);
/* Y (rows x w) = op(A) X: trans = 0 -> A X (Alg. 2 S4), 1 -> A^T X (S2),
 * with the handle's CSR or dense A.  w >= 1 (any width). */
tsvd_status tsvd_dbg_apply(tsvd_t h, int trans, const double* X, int64_t ldx,
                           double* Y, int64_t ldy, int w);
/* CholeskyQR2 in place (Alg. 4): Y (q x w, ld) -> Q, R (w x w row-major).
 * Returns TSVD_WARN_FALLBACK if the CGS2 fallback produced the result. */
tsvd_status tsvd_dbg_cholqr2(double* Y, int64_t q, int w, int64_t ld,
                             double* R, uint64_t seed, void* stream);
/* CGS-CQR2 (Alg. 5): Y (q x w) against P (q x s); both inside ONE row-major
 * buffer `basis` with leading dimension ld: P = columns [0, s), Y = columns
 * [s, s+w).  Outputs H (s x w), R (w x w) row-major.  TSVD_WARN_FALLBACK as
 * for tsvd_dbg_cholqr2. */
tsvd_status tsvd_dbg_cgs_cqr2(double* basis, int64_t q, int s, int w,
                              int64_t ld, double* H, double* R, uint64_t seed,
                              void* stream);
/* CGS-QR (Alg. 3) in place on Y (q x l, ld) with panels of bq -> R (l x l). */
tsvd_status tsvd_dbg_cgs_qr(double* Y, int64_t q, int l, int64_t ld, int bq,
                            double* R, uint64_t seed, void* stream);
/* Small SVD by one-sided Jacobi on the device (reading R20): B (d x d,
 * row-major) -> Ub (d x d), S (d, descending), Vb (d x d), B = Ub S Vb^T. */
tsvd_status tsvd_dbg_small_svd(const double* B, int d, double* Ub, double* S,
                               double* Vb, int* sweeps /* host, may be NULL */,
                               void* stream);
/* Tall-skinny products used by the passes: C (s x w) = X^T Y with X (q x s,
 * ldx), Y (q x w, ldy) (Alg. 5 S1/S6); and Z (q x w) = beta*Z + alpha*X H
 * with H (s x w, ldh) (Alg. 5 S2/S7, restart, outputs). */
tsvd_status tsvd_dbg_gemm_tn(const double* X, int64_t ldx, const double* Y,
                             int64_t ldy, int64_t q, int s, int w, double* C,
                             void* stream);
tsvd_status tsvd_dbg_gemm_nn(const double* X, int64_t ldx, const double* H,
                             int64_t ldh, double* Z, int64_t ldz, int64_t q,
                             int s, int w, double alpha, double beta,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TSVD_H */
