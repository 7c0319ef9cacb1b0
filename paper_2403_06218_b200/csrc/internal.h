// Internal declarations shared by the CUDA translation units of libtsvd.
// Nothing here crosses the C ABI (include/tsvd.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>
#include <string>
#include <vector>

#include "tsvd.h"

namespace tsvd {

// ---------------------------------------------------------------- errors --
struct Error {
  tsvd_status code;
  std::string msg;
};

#define TSVD_CUDA(call)                                                     \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      throw ::tsvd::Error{e_ == cudaErrorMemoryAllocation ? TSVD_ENOMEM     \
                                                          : TSVD_ECUDA,     \
                          std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// every kernel launch site ends with TSVD_CHECK_LAUNCH(): it also counts
// launches for tsvd_info.launches / bench.py's gpu_launches.
extern std::atomic<int64_t> g_launches;
#define TSVD_CHECK_LAUNCH()                                                 \
  do {                                                                      \
    ::tsvd::g_launches.fetch_add(1, std::memory_order_relaxed);             \
    TSVD_CUDA(cudaGetLastError());                                          \
  } while (0)

// Programmatic dependent launch (Hopper+; TSVD_PDL=0 turns it off): the
// hot-path kernels of a solve are launched with programmatic stream
// serialisation, so a kernel's launch and CTA dispatch overlap the tail of
// its predecessor.  Every kernel launched this way starts with pdl_enter():
// griddepcontrol.wait (returns once the predecessor grid has completed and
// its memory is visible -- nothing of the kernel's inputs is read before
// it) and griddepcontrol.launch_dependents (lets the NEXT kernel be launched
// once every CTA of this one has started; its own wait still orders it
// after this grid's completion).  Without the attribute both are no-ops.
extern bool g_pdl;
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  TSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  // (the launch site's TSVD_CHECK_LAUNCH() counts it)
}

// ------------------------------------------------------------ data views --
// Row-major view: element (i, j) at p[i*ld + j].  Row offsets are 64-bit.
struct DMat {
  double* p;
  int64_t rows;
  int cols;
  int64_t ld;
  DMat col(int c0, int w) const { return DMat{p + c0, rows, w, ld}; }
};

struct Csr {  // device CSR (canonical)
  int64_t rows = 0, cols = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  int32_t* colidx = nullptr;
  double* vals = nullptr;
  // load-balancing plan (SpMM): rows longer than kLongRow go to segments
  int64_t nseg = 0;           // number of long-row segments
  int64_t* seg_row = nullptr; // row of each segment
  int64_t* seg_beg = nullptr; // [beg, end) nonzero range of each segment
  int64_t* seg_end = nullptr;
  int32_t* seg_slot = nullptr;   // partial slot (-1: segment covers the whole row)
  int64_t nsplit = 0;            // long rows split into > 1 segment
  int64_t* split_row = nullptr;  // row of each split row
  int32_t* split_first = nullptr;// first partial slot of that row
  int32_t* split_count = nullptr;// number of slots
  int64_t nslots = 0;            // partial slots
  // row-sorted layout (csr_build_plan): after the plan, rowptr/colidx/vals
  // hold the rows in the order [short | medium | long], position p being
  // output row perm[p]; short and medium rows by decreasing length (stable)
  int64_t nshort = 0;            // rows with <= kLongRow nonzeros
  int64_t nmed = 0;              // rows with kLongRow < len <= kMedRow
  int32_t* perm = nullptr;       // output row of each position
  // staged SpMM (spmm.cu, spmm_staged_kernel): rows of equal length L form
  // a bin of consecutive positions (bins in increasing L, L <= kMedRow);
  // per bin: L, row count, first position, first nonzero; and for each of
  // the three chunk sizes NZC = 256 / 128 / 64 (lane groups of 8 / 16 / 32
  // for w <= 16 / 32 / 64) the prefix of chunks over the bins with L <= NZC
  int nbins = 0;
  int64_t* bins = nullptr;       // [nbins][4]: L, count, pos0, nz0
  int64_t* bin_chunk0[3] = {nullptr, nullptr, nullptr};  // [nbins_v + 1]
  int nbins_v[3] = {0, 0, 0};    // bins with L <= NZC_v (a prefix)
  int64_t nchunks[3] = {0, 0, 0};
  int64_t med_gt[3] = {0, 0, 0}; // medium rows longer than NZC_v (warp-per-row path)
};



// ---------------------------------------------------------- kernel entry --
// All launchers enqueue on ctx-independent stream `st`.
void launch_philox_normal(double* out, int64_t q, int w, int64_t ld, uint64_t seed,
                          uint64_t draw, int64_t row0, int64_t q_total, cudaStream_t st);
void launch_philox_words(const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                         int64_t count, cudaStream_t st);

// SpMM: Y (A.rows x w) = A X, w <= 32 per call (callers chunk wider blocks).
void launch_spmm(const Csr& A, const double* X, int64_t ldx, double* Y, int64_t ldy, int w,
                 double* part, cudaStream_t st);
void launch_spmm_wide(const Csr& A, const double* X, int64_t ldx, double* Y, int64_t ldy,
                      int w, double* part, cudaStream_t st);

// CSR transpose on the device (stable: rows of A^T list original rows in
// increasing order).  Allocates T's arrays.
// Device memory of the library: stream-ordered allocations from the
// device's default memory pool, whose release threshold is raised at first
// use so blocks freed by one handle are reused by the next (no cudaMalloc /
// OS round trip per handle); tsvd_trim_memory() returns them.
void* dmalloc(size_t bytes, cudaStream_t st);
void set_allocator(tsvd_alloc_fn a, tsvd_free_fn f, void* ctx);  // tsvd_set_allocator
void dfree(void* p, cudaStream_t st);
template <class T> inline void dmalloc_t(T** p, size_t count, cudaStream_t st) {
  *p = (T*)dmalloc(count * sizeof(T), st);
}
void csr_transpose(const Csr& A, Csr& T, cudaStream_t st);
void csr_build_plan(Csr& A, const int64_t* host_rowptr, cudaStream_t st);
// the plan built on the device (default; the host plan when the staged SpMM
// needs its length bins)
void csr_plan(Csr& A, cudaStream_t st);
void csr_free(Csr& A, cudaStream_t st);
// rows [r0, r1) of a canonical, unplanned CSR as their own planned CSR
void csr_slice_rows(const Csr& A, int64_t r0, int64_t r1, Csr& P, cudaStream_t st);
// device validation of a CSR: 0 if canonical; bits: 1 bad row bounds, 2
// unsorted or duplicate columns in a row (canonicalisable), 4 rowptr[0] != 0
// or rowptr[rows] != nnz, 8 column index out of range
int csr_validate_device(const Csr& A, cudaStream_t st);
// sort each row's columns and sum duplicates (stable order), in place; the
// row pointer is rewritten, nnz may shrink
void csr_canonicalize(Csr& A, cudaStream_t st);

// -------------------------------------------------- tall-skinny products --
// gemm_tn: C (s x w, ldc) = X^T Y  (X: q x s, Y: q x w, both row-major).
// Split over rows into partial sums reduced in a fixed order; part: workspace
// of tn_part_size(q, s) doubles.
size_t tn_part_size(int64_t q, int s);
void gemm_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t q, int s,
             int w, double* C, int64_t ldc, double* part, cudaStream_t st);
// gemm_nn: Z (q x w) = alpha X H + beta Y T   (H: s x w; T: w x w upper
// triangular, optional = identity; Y optional when beta == 0; Z may alias Y).
// gram != null: per-CTA partial Gram Z^T Z (w x w) at gram[cta*w*w] for
// nn_ctas(q, w) CTAs.
int nn_ctas(int64_t q, int w);
// part/part_cap (doubles): optional scratch for split-K partials of plain
// products (beta = 0, no T/gram) with few row tiles; nullptr disables the split.
// X[:, :w] <- X[:, :s] H (s x w, w <= min(s, 128)) in place, one pass over
// X (row-local product; ts.cu).  Returns false when the shape / alignment
// is not supported (the caller stages through scratch instead).
bool gemm_nn_out_inplace(double* X, int64_t ldx, const double* H, int64_t ldh, int64_t q, int s,
                         int w, cudaStream_t st);
void gemm_nn(const double* X, int64_t ldx, const double* H, int64_t ldh, const double* Y,
             int64_t ldy, const double* T, double* Z, int64_t ldz, int64_t q, int s, int w,
             double alpha, double beta, double* gram, cudaStream_t st, double* part = nullptr,
             size_t part_cap = 0);

// small (single-CTA) finalisers (small.cu)
// W = sum of np partial (w x w) Grams; L = chol(W), T = L^{-T}; flag |= breakdown.
void chol_finalize(const double* gram, int np, int w, double* L, double* T, int* flag,
                   cudaStream_t st);
// Lbar = chol(Wbar), Tbar = Lbar^{-T}; R = Lbar^T Lprev^T; H (s x w) += Hbar Lprev^T.
void chol2_finalize(const double* gram, int np, int w, const double* Lprev, double* L2,
                    double* T2, double* R, double* H, const double* Hbar, int s, int* flag,
                    cudaStream_t st);
// W = the same fixed-order sum of np Gram partials the finalisers form (for
// the all-reduce of the multi-GPU path; then finalise with np = 1)
void gram_reduce(const double* gram, int np, int w, double* Wred, cudaStream_t st);
// out[i] = sum_p part[p*count + i], fixed order
void reduce_partials(const double* part, int nparts, int64_t count, double* out,
                     cudaStream_t st);

// BCGS-PIP+ pass finaliser (reading R34): from C = [H; W] ((s+w) x w):
// L = chol(W - H^T H) (flag |= breakdown), T = L^{-T}, Hp = H T; with L1:
// R = L^T L1^T and (Hout != null) Hout = H1 + H L1^T
void pip_finalize(const double* C, int s, int w, double* L, double* T, double* Hp, int* flag,
                  const double* L1, double* R, const double* H1, double* Hout, cudaStream_t st);
// C = alpha op(A) op(B) + beta C on small row-major matrices (fixed order)
void small_gemm(const double* A, int lda, bool ta, const double* B, int ldb, bool tb, double* C,
                int ldc, int m, int n, int k, double alpha, double beta, cudaStream_t st);

// small helpers
void copy_block(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                int cols, bool transpose, cudaStream_t st);
void fill_zero(double* p, int64_t n, cudaStream_t st);

// CGS2 column finalize (fallback path): see blocks.cu
void cgs2_col_finalize(const double* c1, const double* c2, int nb, const double* gram_y,
                       const double* gram_orig, double tau, double* coef_out, double* nrm_out,
                       int* dependent, cudaStream_t st);
void scale_column(double* col, int64_t q, int64_t ld, const double* nrm, cudaStream_t st);

// one-sided Jacobi SVD of a d x d row-major B -> Ub, S (desc), Vb (row-major)
void small_svd(const double* B, int d, double* Ub, double* S, double* Vb, double* work,
               cudaStream_t st);
size_t small_svd_work(int d);
// the same SVD when only Vbar[:, :nv] is needed (LancSVD): the Jacobi sweeps
// skip V, Vbar[:, :nv] = B^T Ubar[:, :nv] / sigma afterwards; the device word
// small_svd_top_ok_dev is 0 when sigma_nv < 1e-3 sigma_1 (then rerun
// small_svd).  part: gemm_tn workspace of tn_part_size(d, d) doubles.
// hog_smem > 0: the Jacobi CTAs request that many bytes of (unused) dynamic
// shared memory, so no streaming-pass CTA shares their SMs while the SVD
// runs beside other work (solvers.cu).
void small_svd_top(const double* B, int d, int nv, double* Ub, double* S, double* Vb,
                   double* work, double* part, cudaStream_t st, int hog_smem = 0);
const unsigned* small_svd_top_ok_dev(const double* work, int d);
int small_svd_sweeps(const double* work, int d);  // sweeps of the last small_svd (syncs)
// device word holding the sweep count of the last small_svd (read together
// with rho once per cycle); a count equal to small_svd_max_sweeps() means the
// sweep cap was hit before the rotation test passed (not converged)
const unsigned* small_svd_sweeps_dev(const double* work, int d);
int small_svd_max_sweeps();
constexpr int kSmallSvdMaxD = 1536;  // largest d the device Jacobi SVD takes

// rho_i = || Rbar * Vb[(k-1)b:kb, i] || / S[0] for i < cnt
void lanczos_rho(const double* Rbar, int b, const double* Vb, int d, const double* S, int cnt,
                 double* rho, cudaStream_t st);
// thick restart (N1): B'[:l,:l] = diag(S), B'[l:l+b, :l] = Rbar Vbar[d-b:d, :l]
void thick_arrow(const double* Rbar, int b, const double* Vb, int d, const double* S, int l,
                 double* B, cudaStream_t st);

// sign normalisation (reading R28): sgn[i] = sign of the largest-|.| entry of
// V[:, i] (lowest index on ties); flip_columns multiplies columns by sgn.
size_t col_signs_work(int r, int world);
double* col_signs_local(const double* V, int64_t n, int64_t ldv, int r, int64_t row0,
                        double* work, cudaStream_t st);
void col_signs_final(const double* all, int world, int r, double* sgn, cudaStream_t st);
void flip_columns(double* M, int64_t rows, int64_t ld, int r, const double* sgn,
                  cudaStream_t st);

}  // namespace tsvd
