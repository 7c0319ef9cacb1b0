// extern "C" entry points of include/tsvd.h.  Argument validation, copies
// across the host/device boundary, and exception -> status translation.
#include <algorithm>
#include <mutex>
#include <vector>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ctx.h"

namespace tsvd {
std::atomic<int64_t> g_launches{0};
bool g_pdl = getenv("TSVD_PDL") ? atoi(getenv("TSVD_PDL")) != 0 : false;  // measured: no gain (DESIGN 6)
static thread_local std::string g_last_error;
}  // namespace tsvd

using namespace tsvd;

#define TSVD_API_BEGIN try {
#define TSVD_API_END                                   \
  }                                                    \
  catch (const tsvd::Error& e) {                       \
    tsvd::g_last_error = e.msg;                        \
    return e.code;                                     \
  }                                                    \
  catch (const std::bad_alloc&) {                      \
    return TSVD_ENOMEM;                                \
  }                                                    \
  catch (...) {                                        \
    return TSVD_ECUDA;                                 \
  }

// Pinned host words for the per-cycle flag / sweep read-backs, handed out
// from a process-wide arena: cudaMallocHost / cudaFreeHost per handle
// synchronise the device (and cost milliseconds on a busy host).
static std::mutex g_pin_mu;
static std::vector<int*> g_pin_free;
static int* pinned_words() {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_free.empty()) {
    int* blk = nullptr;
    TSVD_CUDA(cudaMallocHost(&blk, 64 * 8 * sizeof(int)));  // 64 slots of 8 ints, never freed
    for (int i = 0; i < 64; ++i) g_pin_free.push_back(blk + 8 * i);
  }
  int* p = g_pin_free.back();
  g_pin_free.pop_back();
  return p;
}
static void pinned_words_free(int* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

static tsvd_status init_ctx(tsvd_ctx* c) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return TSVD_ECUDA;
  }
  TSVD_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  c->own_stream = true;
  c->dflags = (int*)dmalloc(4 * sizeof(int), c->st);  // stream-ordered pool, no device sync
  c->hflags = pinned_words();
  return TSVD_OK;
}

static void destroy_ctx(tsvd_ctx* c) {
  if (!c) return;
  // side streams first: after an error inside a solve the forked SVD or a
  // reduction may still be running on buffers freed below
  if (c->svd_st) cudaStreamSynchronize(c->svd_st);
  if (c->comm_st) cudaStreamSynchronize(c->comm_st);
  if (c->copy_st) cudaStreamSynchronize(c->copy_st);
  if (c->st) cudaStreamSynchronize(c->st);
  csr_free(c->A, c->st);
  csr_free(c->AT, c->st);
  for (auto& P : c->ATp) csr_free(P, c->st);
  for (auto e : c->comm_ev) cudaEventDestroy(e);
  if (c->comm_st) cudaStreamDestroy(c->comm_st);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->svd_st) cudaStreamDestroy(c->svd_st);
  if (c->svd_fork) cudaEventDestroy(c->svd_fork);
  if (c->svd_join) cudaEventDestroy(c->svd_join);
  if (c->copy_ev) cudaEventDestroy(c->copy_ev);
  dfree(c->Ad, c->st);
  free_bufs(*c);
  prof_release(*c);
  comm_destroy(*c);
  if (c->dflags) dfree(c->dflags, c->st);
  pinned_words_free(c->hflags);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
}

extern "C" {

const char* tsvd_strerror(tsvd_status s) {
  switch (s) {
    case TSVD_OK: return "ok";
    case TSVD_WARN_NOTCONV: return "not converged within maxit (results retrievable)";
    case TSVD_WARN_FALLBACK: return "Cholesky breakdown: CGS2 fallback used (P:275)";
    case TSVD_WARN_SVD: return "device Jacobi SVD hit its sweep cap (results retrievable)";
    case TSVD_EINVAL: return "invalid argument";
    case TSVD_ESHAPE: return "invalid shape";
    case TSVD_ENOMEM: return "device out of memory";
    case TSVD_ECUDA: return "CUDA error or no usable device";
    case TSVD_ENCCL: return "NCCL unavailable or failed";
    case TSVD_ESTATE: return "invalid state (no results yet)";
    default: return "unknown status";
  }
}

const char* tsvd_last_error(void) { return tsvd::g_last_error.c_str(); }

// Build the CSR part of a handle whose local/global geometry is already set:
// c->m local rows, c->ng columns.  Validates, uploads, transposes, plans.
// TSVD_TIMING=1: create-time phases on stderr (development)
struct PhaseClock {
  bool on = getenv("TSVD_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[tsvd create] %-12s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

static tsvd_status setup_csr(tsvd_ctx* c, int64_t nnz, const int64_t* rowptr,
                             const int32_t* colidx, const double* vals, int mem_kind) {
  PhaseClock clk;
  const int64_t m = c->m, n = c->ng;
  Csr& A = c->A;
  A.rows = m;
  A.cols = n;
  A.nnz = nnz;
  const cudaMemcpyKind kind = mem_kind == TSVD_DEVICE ? cudaMemcpyDeviceToDevice
                                                      : cudaMemcpyHostToDevice;
  if (mem_kind != TSVD_DEVICE) {
    // row pointer checked here (O(m)); the column indices on the device below
    if (rowptr[0] != 0 || rowptr[m] != nnz) return TSVD_EINVAL;
    for (int64_t i = 0; i < m; ++i)
      if (rowptr[i + 1] < rowptr[i]) return TSVD_EINVAL;
  }
  dmalloc_t(&A.rowptr, m + 1, c->st);
  dmalloc_t(&A.colidx, std::max<int64_t>(1, nnz), c->st);
  dmalloc_t(&A.vals, std::max<int64_t>(1, nnz), c->st);
  TSVD_CUDA(cudaMemcpyAsync(A.rowptr, rowptr, (m + 1) * sizeof(int64_t), kind, c->st));
  if (nnz > 0) {
    TSVD_CUDA(cudaMemcpyAsync(A.colidx, colidx, nnz * sizeof(int32_t), kind, c->st));
    TSVD_CUDA(cudaMemcpyAsync(A.vals, vals, nnz * sizeof(double), kind, c->st));
  }
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  clk.lap("upload", c->st);
  const int bad = csr_validate_device(A, c->st);  // warp per row, exact
  clk.lap("validate", c->st);
  if (bad & ~2) return TSVD_EINVAL;               // bounds / out-of-range columns
  if (bad & 2) csr_canonicalize(A, c->st);        // unsorted or duplicates: canonicalise
  csr_transpose(A, c->AT, c->st);
  clk.lap("transpose", c->st);
  if (c->world > 1) {  // n-shard pieces of CSR(A_g^T) for the pipelined reduce-scatter
    c->ATp.resize(c->world);
    for (int g = 0; g < c->world; ++g) {
      const int64_t r0 = std::min<int64_t>(n, (int64_t)g * c->nsh);
      const int64_t r1 = std::min<int64_t>(n, r0 + c->nsh);
      csr_slice_rows(c->AT, r0, r1, c->ATp[g], c->st);
    }
  }
  csr_plan(A, c->st);
  clk.lap("plan A", c->st);
  csr_plan(c->AT, c->st);
  clk.lap("plan A^T", c->st);
  return TSVD_OK;
}

// Dense rows (c->m x c->ng), row-major lda or (single GPU) column-major.
static tsvd_status setup_dense(tsvd_ctx* c, const double* Ain, int64_t lda, int layout,
                               int mem_kind) {
  const int64_t m = c->m, n = c->ng;
  c->dense = true;
  c->lda = n;
  dmalloc_t(&c->Ad, (size_t)std::max<int64_t>(1, m) * n, c->st);
  const cudaMemcpyKind kind = mem_kind == TSVD_DEVICE ? cudaMemcpyDeviceToDevice
                                                      : cudaMemcpyHostToDevice;
  if (layout == TSVD_ROW_MAJOR) {
    if (m > 0)
      TSVD_CUDA(cudaMemcpy2DAsync(c->Ad, n * sizeof(double), Ain, lda * sizeof(double),
                                  n * sizeof(double), m, kind, c->st));
  } else {
    // column-major input: upload as an n x m row-major block, transpose on device
    double* tmp;
    dmalloc_t(&tmp, (size_t)m * n, c->st);
    TSVD_CUDA(cudaMemcpy2DAsync(tmp, m * sizeof(double), Ain, lda * sizeof(double),
                                m * sizeof(double), n, kind, c->st));
    copy_block(tmp, m, c->Ad, n, m, (int)n, true, c->st);
    TSVD_CUDA(cudaStreamSynchronize(c->st));
    dfree(tmp, c->st);
  }
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  return TSVD_OK;
}

static void set_single(tsvd_ctx* c, int64_t m, int64_t n) {
  c->m = c->mg = m;
  c->n = c->ng = c->nsh = n;
  c->m0 = c->n0 = 0;
  c->world = 1;
  c->rank = 0;
}

static tsvd_status set_dist(tsvd_ctx* c, const tsvd_dist* d) {
  if (!d || d->world < 1 || d->rank < 0 || d->rank >= d->world || (!d->nccl_id && !d->loopback))
    return TSVD_EINVAL;
  if (d->m_global < d->n_global) return TSVD_ESHAPE;
  if (d->row_begin < 0 || d->row_end < d->row_begin || d->row_end > d->m_global)
    return TSVD_EINVAL;
  if (d->n_global < 1 || d->n_global >= (int64_t)INT32_MAX) return TSVD_ESHAPE;
  c->world = d->world;
  c->rank = d->rank;
  c->mg = d->m_global;
  c->ng = d->n_global;
  c->m = d->row_end - d->row_begin;
  c->m0 = d->row_begin;
  c->nsh = (c->ng + c->world - 1) / c->world;
  c->n0 = std::min<int64_t>(c->ng, (int64_t)c->rank * c->nsh);
  c->n = std::min<int64_t>(c->ng, c->n0 + c->nsh) - c->n0;
  return TSVD_OK;
}

#define TSVD_CREATE_CATCH                        \
  catch (const tsvd::Error& e) {                 \
    tsvd::g_last_error = e.msg;                  \
    destroy_ctx(c);                              \
    return e.code;                               \
  }                                              \
  catch (...) {                                  \
    destroy_ctx(c);                              \
    return TSVD_ECUDA;                           \
  }

tsvd_status tsvd_create_csr(tsvd_t* h, int64_t m, int64_t n, int64_t nnz,
                            const int64_t* rowptr, const int32_t* colidx, const double* vals,
                            int mem_kind) {
  if (!h || !rowptr || (nnz > 0 && (!colidx || !vals)) || m < 0 || n < 1 || nnz < 0)
    return TSVD_EINVAL;
  if (m < n) return TSVD_ESHAPE;
  if (n >= (int64_t)INT32_MAX || m >= (int64_t)INT32_MAX) return TSVD_ESHAPE;
  *h = nullptr;
  tsvd_ctx* c = new tsvd_ctx();
  try {
    tsvd_status s = init_ctx(c);
    if (s == TSVD_OK) {
      set_single(c, m, n);
      s = setup_csr(c, nnz, rowptr, colidx, vals, mem_kind);
    }
    if (s != TSVD_OK) {
      destroy_ctx(c);
      return s;
    }
    *h = c;
    return TSVD_OK;
  }
  TSVD_CREATE_CATCH
}

tsvd_status tsvd_create_dense(tsvd_t* h, int64_t m, int64_t n, const double* Ain, int64_t lda,
                              int layout, int mem_kind) {
  if (!h || !Ain || m < 1 || n < 1) return TSVD_EINVAL;
  if (m < n) return TSVD_ESHAPE;
  if (layout == TSVD_ROW_MAJOR ? lda < n : lda < m) return TSVD_EINVAL;
  if (n >= (int64_t)INT32_MAX) return TSVD_ESHAPE;
  *h = nullptr;
  tsvd_ctx* c = new tsvd_ctx();
  try {
    tsvd_status s = init_ctx(c);
    if (s == TSVD_OK) {
      set_single(c, m, n);
      s = setup_dense(c, Ain, lda, layout, mem_kind);
    }
    if (s != TSVD_OK) {
      destroy_ctx(c);
      return s;
    }
    *h = c;
    return TSVD_OK;
  }
  TSVD_CREATE_CATCH
}

static void join_comm(tsvd_ctx* c, const tsvd_dist* d) {
  if (d->loopback)
    loop_join(*c, static_cast<LoopGroup*>(d->loopback), d->rank);
  else
    comm_init(*c, d->nccl_id, d->rank, d->world);
}

tsvd_status tsvd_loopback_create(int world, void** group) {
  if (!group || world < 1 || world > kLoopMaxWorld) return TSVD_EINVAL;
  TSVD_API_BEGIN
  *group = loop_group_create(world);
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_loopback_destroy(void* group) {
  if (!group) return TSVD_EINVAL;
  loop_group_destroy(static_cast<LoopGroup*>(group));
  return TSVD_OK;
}

tsvd_status tsvd_create_csr_dist(tsvd_t* h, const tsvd_dist* dist, int64_t nnz,
                                 const int64_t* rowptr, const int32_t* colidx,
                                 const double* vals, int mem_kind) {
  if (!h || !rowptr || (nnz > 0 && (!colidx || !vals)) || nnz < 0) return TSVD_EINVAL;
  *h = nullptr;
  tsvd_ctx* c = new tsvd_ctx();
  try {
    tsvd_status s = init_ctx(c);
    if (s == TSVD_OK) s = set_dist(c, dist);
    if (s == TSVD_OK) s = setup_csr(c, nnz, rowptr, colidx, vals, mem_kind);
    if (s == TSVD_OK) join_comm(c, dist);
    if (s != TSVD_OK) {
      destroy_ctx(c);
      return s;
    }
    *h = c;
    return TSVD_OK;
  }
  TSVD_CREATE_CATCH
}

tsvd_status tsvd_create_dense_dist(tsvd_t* h, const tsvd_dist* dist, const double* Ain,
                                   int64_t lda, int mem_kind) {
  if (!h || !dist) return TSVD_EINVAL;
  *h = nullptr;
  tsvd_ctx* c = new tsvd_ctx();
  try {
    tsvd_status s = init_ctx(c);
    if (s == TSVD_OK) s = set_dist(c, dist);
    if (s == TSVD_OK && (c->m > 0 && (!Ain || lda < c->ng))) s = TSVD_EINVAL;
    if (s == TSVD_OK) s = setup_dense(c, Ain, lda, TSVD_ROW_MAJOR, mem_kind);
    if (s == TSVD_OK) join_comm(c, dist);
    if (s != TSVD_OK) {
      destroy_ctx(c);
      return s;
    }
    *h = c;
    return TSVD_OK;
  }
  TSVD_CREATE_CATCH
}

tsvd_status tsvd_nccl_unique_id(void* out128) {
  if (!out128) return TSVD_EINVAL;
  TSVD_API_BEGIN
  nccl_unique_id(out128);
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_partition_rows(const int64_t* rowptr, int64_t m, int world, int64_t* bounds) {
  if (!rowptr || !bounds || m < 0 || world < 1) return TSVD_EINVAL;
  const int64_t nnz = rowptr[m];
  bounds[0] = 0;
  int64_t r = 0;
  for (int g = 1; g < world; ++g) {
    const int64_t target = (nnz * g + world - 1) / world;  // first row whose prefix >= target
    while (r < m && rowptr[r] < target) ++r;
    int64_t b = r;  // nearest row boundary to the target prefix
    if (r > bounds[g - 1] && target - rowptr[r - 1] < rowptr[r] - target) b = r - 1;
    bounds[g] = std::max(bounds[g - 1], b);
  }
  bounds[world] = m;
  return TSVD_OK;
}

tsvd_status tsvd_set_stream(tsvd_t h, void* stream) {
  if (!h) return TSVD_EINVAL;
  TSVD_API_BEGIN
  TSVD_CUDA(cudaStreamSynchronize(h->st));
  if (h->own_stream) cudaStreamDestroy(h->st);
  h->st = (cudaStream_t)stream;  // NULL = legacy default stream
  h->own_stream = false;
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_set_seed(tsvd_t h, uint64_t seed) {
  if (!h) return TSVD_EINVAL;
  h->seed = seed;
  return TSVD_OK;
}

tsvd_status tsvd_set_krylov_dim(tsvd_t h, int d) {
  if (!h || d < 0) return TSVD_EINVAL;
  h->krylov_d = d;
  return TSVD_OK;
}

tsvd_status tsvd_trim_memory(size_t keep_bytes) {
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) {
    cudaGetLastError();
    return TSVD_ECUDA;
  }
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemPoolTrimTo(pool, keep_bytes) != cudaSuccess) {
    cudaGetLastError();
    return TSVD_ECUDA;
  }
  return TSVD_OK;
}

tsvd_status tsvd_set_allocator(tsvd_alloc_fn alloc, tsvd_free_fn free_, void* ctx) {
  if ((alloc == nullptr) != (free_ == nullptr)) return TSVD_EINVAL;
  set_allocator(alloc, free_, ctx);
  return TSVD_OK;
}

tsvd_status tsvd_set_thick_restart(tsvd_t h, int keep) {
  if (!h || keep < 0) return TSVD_EINVAL;
  h->thick_keep = keep;
  return TSVD_OK;
}

tsvd_status tsvd_set_output_mode(tsvd_t h, int mode) {
  if (!h || mode < TSVD_OUT_AUTO || mode > TSVD_OUT_INPLACE) return TSVD_EINVAL;
  h->out_mode = mode;
  return TSVD_OK;
}

tsvd_status tsvd_set_graphs(tsvd_t h, int on) {
  if (!h) return TSVD_EINVAL;
  TSVD_API_BEGIN
  if (!on) cycle_graph_reset(*h);
  h->graphs = on != 0;
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_set_ortho(tsvd_t h, int ortho) {
  if (!h || (ortho != TSVD_ORTHO_CGS_CQR2 && ortho != TSVD_ORTHO_BCGS_PIP2)) return TSVD_EINVAL;
  h->ortho = ortho;
  return TSVD_OK;
}

tsvd_status tsvd_set_qr_block(tsvd_t h, int b_qr) {
  if (!h || b_qr < 1 || b_qr > 32) return TSVD_EINVAL;
  h->b_qr = b_qr;
  return TSVD_OK;
}

tsvd_status tsvd_set_start(tsvd_t h, const double* block, int64_t rows, int64_t cols,
                           int64_t ld, int mem_kind) {
  if (!h) return TSVD_EINVAL;
  if (!block) {
    h->start.clear();
    h->start_rows = h->start_cols = 0;
    return TSVD_OK;
  }
  if (rows < 1 || cols < 1 || ld < cols) return TSVD_EINVAL;
  TSVD_API_BEGIN
  h->start.resize((size_t)rows * cols);
  TSVD_CUDA(cudaMemcpy2D(h->start.data(), cols * sizeof(double), block, ld * sizeof(double),
                         cols * sizeof(double), rows,
                         mem_kind == TSVD_DEVICE ? cudaMemcpyDeviceToHost
                                                 : cudaMemcpyHostToHost));
  h->start_rows = rows;
  h->start_cols = cols;
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_block_lanczos(tsvd_t h, int r, int b, double tol, int maxit) {
  if (!h) return TSVD_EINVAL;
  TSVD_API_BEGIN
  return lanczos_solve(*h, r, b, tol, maxit);
  TSVD_API_END
}

tsvd_status tsvd_block_lanczos_threshold(tsvd_t h, double tau, int b, double tol, int maxit,
                                         int r_max, int* r_out) {
  if (!h) return TSVD_EINVAL;
  TSVD_API_BEGIN
  return lanczos_threshold(*h, tau, b, tol, maxit, r_max, r_out);
  TSVD_API_END
}

tsvd_status tsvd_rsvd(tsvd_t h, int r, int p, int q) {
  if (!h) return TSVD_EINVAL;
  TSVD_API_BEGIN
  return rsvd_solve(*h, r, p, q);
  TSVD_API_END
}

tsvd_status tsvd_get(tsvd_t h, double* U, int64_t ldu, double* S, double* V, int64_t ldv,
                     int mem_kind) {
  if (!h) return TSVD_EINVAL;
  if (!h->have) return TSVD_ESTATE;
  const int r = h->r;
  if ((U && ldu < r) || (V && ldv < r)) return TSVD_EINVAL;
  TSVD_API_BEGIN
  const cudaMemcpyKind k = mem_kind == TSVD_DEVICE ? cudaMemcpyDeviceToDevice
                                                   : cudaMemcpyDeviceToHost;
  // to the host with both U and V wanted: V on a second stream (after the
  // solve's work on h->st), so the two copies use two copy engines
  cudaStream_t vst = h->st;
  static const bool two_streams =
      getenv("TSVD_GET_2STREAM") ? atoi(getenv("TSVD_GET_2STREAM")) != 0 : true;
  if (two_streams && U && V && k == cudaMemcpyDeviceToHost) {
    if (!h->copy_st) {
      TSVD_CUDA(cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking));
      TSVD_CUDA(cudaEventCreateWithFlags(&h->copy_ev, cudaEventDisableTiming));
    }
    TSVD_CUDA(cudaEventRecord(h->copy_ev, h->st));
    TSVD_CUDA(cudaStreamWaitEvent(h->copy_st, h->copy_ev, 0));
    vst = h->copy_st;
  }
  if (V)
    TSVD_CUDA(cudaMemcpy2DAsync(V, ldv * sizeof(double), h->V, h->ldV * sizeof(double),
                                r * sizeof(double), h->n, k, vst));
  if (U)
    TSVD_CUDA(cudaMemcpy2DAsync(U, ldu * sizeof(double), h->U, h->ldU * sizeof(double),
                                r * sizeof(double), h->m, k, h->st));
  if (S) TSVD_CUDA(cudaMemcpyAsync(S, h->S, r * sizeof(double), k, h->st));
  if (vst != h->st) TSVD_CUDA(cudaStreamSynchronize(vst));
  TSVD_CUDA(cudaStreamSynchronize(h->st));
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_residuals(tsvd_t h, double* e, double* rel) {
  if (!h) return TSVD_EINVAL;
  if (!h->have) return TSVD_ESTATE;
  TSVD_API_BEGIN
  residuals(*h, e, rel);
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_get_info(tsvd_t h, tsvd_info* out) {
  if (!h || !out) return TSVD_EINVAL;
  *out = h->info;
  return TSVD_OK;
}

tsvd_status tsvd_get_rho(tsvd_t h, double* rho) {
  if (!h || !rho) return TSVD_EINVAL;
  if (!h->have || h->rho.empty()) return TSVD_ESTATE;
  std::copy(h->rho.begin(), h->rho.end(), rho);
  return TSVD_OK;
}

tsvd_status tsvd_set_profiling(tsvd_t h, int on) {
  if (!h) return TSVD_EINVAL;
  h->prof_mask = on != 0 ? (1u << TSVD_NPROF) - 1u : 0u;
  h->prof_on = h->prof_mask != 0;
  return TSVD_OK;
}

tsvd_status tsvd_set_profiling_mask(tsvd_t h, unsigned mask) {
  if (!h) return TSVD_EINVAL;
  h->prof_mask = mask & ((1u << TSVD_NPROF) - 1u);
  h->prof_on = h->prof_mask != 0;
  return TSVD_OK;
}

tsvd_status tsvd_get_profile(tsvd_t h, tsvd_prof_entry* out) {
  if (!h || !out) return TSVD_EINVAL;
  TSVD_API_BEGIN
  TSVD_CUDA(cudaStreamSynchronize(h->st));
  prof_harvest(*h);
  for (int i = 0; i < TSVD_NPROF; ++i) out[i] = h->prof[i];
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_reset_profile(tsvd_t h) {
  if (!h) return TSVD_EINVAL;
  TSVD_API_BEGIN
  TSVD_CUDA(cudaStreamSynchronize(h->st));
  prof_harvest(*h);
  for (int i = 0; i < TSVD_NPROF; ++i) {
    const char* nm = h->prof[i].name;
    h->prof[i] = tsvd_prof_entry{};
    h->prof[i].name = nm;
  }
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_destroy(tsvd_t h) {
  if (!h) return TSVD_EINVAL;
  destroy_ctx(h);
  return TSVD_OK;
}

// ------------------------------------------------------------------ debug --
static tsvd_ctx* dbg_ctx(void* stream) {
  static thread_local tsvd_ctx* c = nullptr;
  if (!c) {
    c = new tsvd_ctx();
    TSVD_CUDA(cudaMalloc(&c->dflags, 4 * sizeof(int)));
    TSVD_CUDA(cudaMallocHost(&c->hflags, 8 * sizeof(int)));
  }
  c->st = (cudaStream_t)stream;
  c->own_stream = false;
  return c;
}

tsvd_status tsvd_dbg_philox(double* out, int64_t q, int w, int64_t ld, uint64_t seed,
                            uint64_t draw, int64_t row0, int64_t q_total, void* stream) {
  if (!out || q < 0 || w < 1 || ld < w) return TSVD_EINVAL;
  TSVD_API_BEGIN
  launch_philox_normal(out, q, w, ld, seed, draw, row0, q_total, (cudaStream_t)stream);
  TSVD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_philox_words(const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                                  int64_t count, void* stream) {
  if (!ctr || !key || !out || count < 0) return TSVD_EINVAL;
  TSVD_API_BEGIN
  launch_philox_words(ctr, key, out, count, (cudaStream_t)stream);
  TSVD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_apply(tsvd_t h, int trans, const double* X, int64_t ldx, double* Y,
                           int64_t ldy, int w) {
  if (!h || !X || !Y || w < 1 || ldx < w || ldy < w) return TSVD_EINVAL;
  TSVD_API_BEGIN
  apply(*h, trans != 0, X, ldx, Y, ldy, w);
  TSVD_CUDA(cudaStreamSynchronize(h->st));
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_cholqr2(double* Y, int64_t q, int w, int64_t ld, double* R, uint64_t seed,
                             void* stream) {
  if (!Y || !R || q < 1 || w < 1 || w > 32 || ld < w) return TSVD_EINVAL;
  TSVD_API_BEGIN
  tsvd_ctx* c = dbg_ctx(stream);
  c->seed = seed;
  c->draw_next = 1;
  const int fb = cholqr2(*c, Y, q, w, ld, R);
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  return fb ? TSVD_WARN_FALLBACK : TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_cgs_cqr2(double* basis, int64_t q, int s, int w, int64_t ld, double* H,
                              double* R, uint64_t seed, void* stream) {
  if (!basis || !R || (s > 0 && !H) || q < 1 || s < 0 || w < 1 || w > 32 || ld < s + w)
    return TSVD_EINVAL;
  TSVD_API_BEGIN
  tsvd_ctx* c = dbg_ctx(stream);
  c->seed = seed;
  c->draw_next = 1;
  const int fb = cgs_cqr2(*c, basis, q, s, w, ld, H, R);
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  return fb ? TSVD_WARN_FALLBACK : TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_cgs_qr(double* Y, int64_t q, int l, int64_t ld, int bq, double* R,
                            uint64_t seed, void* stream) {
  if (!Y || !R || q < 1 || l < 1 || bq < 1 || bq > 32 || ld < l) return TSVD_EINVAL;
  TSVD_API_BEGIN
  tsvd_ctx* c = dbg_ctx(stream);
  c->seed = seed;
  c->draw_next = 1;
  cgs_qr(*c, Y, q, l, ld, bq, R);
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_small_svd(const double* B, int d, double* Ub, double* S, double* Vb,
                               int* sweeps, void* stream) {
  if (!B || !Ub || !S || !Vb || d < 1) return TSVD_EINVAL;
  TSVD_API_BEGIN
  tsvd_ctx* c = dbg_ctx(stream);
  double* work = dbuf(*c, "jacobi_work", small_svd_work(d));
  // development A/B: TSVD_DBG_SVD_TOP = nv runs the Lanczos driver's
  // top-nv path (no rotated V; Vbar[:, :nv] = B^T Ubar / sigma)
  static const int top_nv = getenv("TSVD_DBG_SVD_TOP") ? atoi(getenv("TSVD_DBG_SVD_TOP")) : 0;
  if (top_nv > 0)
    small_svd_top(B, d, std::min(top_nv, d), Ub, S, Vb, work, dbuf(*c, "part_tn", tn_part_size(d, d)), c->st);
  else
    small_svd(B, d, Ub, S, Vb, work, c->st);
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  const int sw = small_svd_sweeps(work, d);
  if (sweeps) *sweeps = sw;
  return sw >= small_svd_max_sweeps() ? TSVD_WARN_SVD : TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_gemm_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy,
                             int64_t q, int s, int w, double* C, void* stream) {
  if (!X || !Y || !C || q < 0 || s < 1 || w < 1) return TSVD_EINVAL;
  TSVD_API_BEGIN
  tsvd_ctx* c = dbg_ctx(stream);
  double* part = dbuf(*c, "part_tn", tn_part_size(q, s));
  gemm_tn(X, ldx, Y, ldy, q, s, w, C, w, part, c->st);
  TSVD_CUDA(cudaStreamSynchronize(c->st));
  return TSVD_OK;
  TSVD_API_END
}

tsvd_status tsvd_dbg_gemm_nn(const double* X, int64_t ldx, const double* H, int64_t ldh,
                             double* Z, int64_t ldz, int64_t q, int s, int w, double alpha,
                             double beta, void* stream) {
  if (!Z || q < 0 || s < 0 || w < 1 || (s > 0 && (!X || !H))) return TSVD_EINVAL;
  TSVD_API_BEGIN
  gemm_nn(X, ldx, H, ldh, Z, ldz, nullptr, Z, ldz, q, s, w, alpha, beta, nullptr,
          (cudaStream_t)stream);
  TSVD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return TSVD_OK;
  TSVD_API_END
}

}  // extern "C"
