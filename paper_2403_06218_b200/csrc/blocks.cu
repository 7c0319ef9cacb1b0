// Building blocks of Sec. 3 on the device, composed from the
// kernels of ts.cu / spmm.cu:
//   cholqr2   Alg. 4  readings R3, R4
//   cgs_cqr2  Alg. 5  readings R4, R5
//   cgs2      P:275 fallback        reading R16
//   cgs_qr    Alg. 3  reading R8
//   apply     A.X / A^T.X (Alg. 1 S1/S3, Alg. 2 S2/S4; dense: Table 1 "*")
//
// Pass structure of CGS-CQR2 on q x w against q x s (each pass reads P once):
//   1 gemm_tn : H     = P^T Y                         (S1)
//   2 gemm_nn : S     = Y - P H,  W = S^T S            (S2, S3)      -> L = chol(W)     (S4)
//   3 gemm_tn : Hbar  = P^T (S L^{-T})                 (S5 fused into S6)
//   4 gemm_nn : S     = S L^{-T} - P Hbar, Wbar = S^T S (S5, S7, S8)  -> Lbar, R, H (S9, S11, S12)
//   5 gemm_nn : Y     = S Lbar^{-T}                    (S10)
// Y itself is only overwritten by pass 5, after the host has seen both
// breakdown flags, so the CGS2 fallback always restarts from the original Y
// exactly as in the oracle (one stream sync per orthogonalisation).
#include <mutex>
#include <unordered_map>

#include <algorithm>

#include "ctx.h"

namespace tsvd {

static void pool_init() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done = true;
}

// Caller-registered allocator (tsvd_set_allocator), process-wide.  Blocks it
// returned are remembered so that they go back to it (and blocks from the
// default pool back to the pool) whatever is registered when they are freed.
static std::mutex g_alloc_mu;
static tsvd_alloc_fn g_alloc = nullptr;
static tsvd_free_fn g_free = nullptr;
static void* g_alloc_ctx = nullptr;
static std::unordered_map<void*, std::pair<tsvd_free_fn, void*>> g_user_blocks;

void set_allocator(tsvd_alloc_fn a, tsvd_free_fn f, void* ctx) {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  g_alloc = a;
  g_free = f;
  g_alloc_ctx = ctx;
}

void* dmalloc(size_t bytes, cudaStream_t st) {
  {
    std::unique_lock<std::mutex> lk(g_alloc_mu);
    if (g_alloc) {
      tsvd_alloc_fn a = g_alloc;
      tsvd_free_fn f = g_free;
      void* ctx = g_alloc_ctx;
      lk.unlock();
      void* p = a(bytes ? bytes : 8, (void*)st, ctx);
      if (!p) throw Error{TSVD_ENOMEM, "registered allocator returned NULL"};
      lk.lock();
      g_user_blocks[p] = {f, ctx};
      return p;
    }
  }
  pool_init();
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 8, st);
  if (e == cudaErrorMemoryAllocation) {
    // the pool retains freed blocks (release threshold raised in pool_init);
    // blocks of other sizes (e.g. create-time transposition temporaries) can
    // not serve a large request, so hand them back to the system and retry
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaStreamSynchronize(st) == cudaSuccess && cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
    cudaGetLastError();
    e = cudaMallocAsync(&p, bytes ? bytes : 8, st);
  }
  TSVD_CUDA(e);
  return p;
}

void dfree(void* p, cudaStream_t st) {
  if (!p) return;
  {
    std::unique_lock<std::mutex> lk(g_alloc_mu);
    auto it = g_user_blocks.find(p);
    if (it != g_user_blocks.end()) {
      auto fc = it->second;
      g_user_blocks.erase(it);
      lk.unlock();
      fc.first(p, (void*)st, fc.second);
      return;
    }
  }
  cudaFreeAsync(p, st);
}

void* buf(Ctx& c, const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 8;
  auto it = c.bufs.find(name);
  if (it != c.bufs.end() && it->second.second >= bytes) return it->second.first;
  if (it != c.bufs.end()) {
    if (c.capturing) throw Error{TSVD_ECUDA, "buffer reallocation inside a graph capture"};
    dfree(it->second.first, c.st);  // stream-ordered: pending work on c.st finishes first
    c.bufs.erase(it);
  }
  if (c.capturing) throw Error{TSVD_ECUDA, "buffer allocation inside a graph capture"};
  void* p = dmalloc(bytes, c.st);
  c.bufs[name] = {p, bytes};
  ++c.bufgen;
  return p;
}

void free_bufs(Ctx& c) {
  for (auto& kv : c.bufs) dfree(kv.second.first, c.st);
  c.bufs.clear();
}

static const char* kProfNames[TSVD_NPROF] = {"apply_A",     "apply_AT",  "ortho_tn",
                                             "ortho_nn",    "ortho_small", "small_svd",
                                             "restart_out", "other",     "ortho_rowT",
                                             "beside_svd"};

static cudaEvent_t pool_get(Ctx& c) {
  if (!c.ev_pool.empty()) {
    cudaEvent_t e = c.ev_pool.back();
    c.ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  TSVD_CUDA(cudaEventCreate(&e));
  return e;
}

// inside a stream capture the records become event-record nodes of the graph
// (external events), so every replay re-records them for the same harvest
static cudaError_t record(Ctx& c, cudaEvent_t e) {
  return c.capturing ? cudaEventRecordWithFlags(e, c.st, cudaEventRecordExternal)
                     : cudaEventRecord(e, c.st);
}

Prof::Prof(Ctx& c_, int cat_, double bytes_, double flops_)
    : c(c_), cat(c_.prof_override >= 0 ? c_.prof_override : cat_), bytes(bytes_), flops(flops_) {
  if (!c.prof_on || !((c.prof_mask >> cat) & 1u)) return;
  a = pool_get(c);
  TSVD_CUDA(record(c, a));
  l0 = g_launches.load();
}

Prof::~Prof() {
  if (!c.prof_on || !a) return;
  cudaEvent_t b = pool_get(c);
  record(c, b);
  c.prof_open.push_back(ProfRec{cat, a, b, g_launches.load() - l0, bytes, flops});
}

void prof_harvest(Ctx& c) {
  for (auto& r : c.prof_open) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    tsvd_prof_entry& e = c.prof[r.cat];
    e.name = kProfNames[r.cat];
    e.calls += 1;
    e.launches += r.launches;
    e.ms += ms;
    e.bytes += r.bytes;
    e.flops += r.flops;
    if (!r.graph_owned) {
      c.ev_pool.push_back(r.a);
      c.ev_pool.push_back(r.b);
    }
  }
  c.prof_open.clear();
  for (int i = 0; i < TSVD_NPROF; ++i) c.prof[i].name = kProfNames[i];
}

void cycle_graph_reset(Ctx& c) {
  CycleGraph& g = c.cyc_graph;
  if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& r : g.prof_recs) {
    c.ev_pool.push_back(r.a);
    c.ev_pool.push_back(r.b);
  }
  g = CycleGraph{};
}

void prof_release(Ctx& c) {
  cycle_graph_reset(c);
  for (auto& r : c.prof_open) {
    if (r.graph_owned) continue;
    c.ev_pool.push_back(r.a);
    c.ev_pool.push_back(r.b);
  }
  c.prof_open.clear();
  for (auto e : c.ev_pool) cudaEventDestroy(e);
  c.ev_pool.clear();
}

// algorithmic traffic of the pass kernels
static double tn_bytes(int64_t q, int s, int w) { return 8.0 * q * (s + w); }
static double nn_bytes(int64_t q, int s, int w, bool readY, bool writeZ) {
  return 8.0 * q * (s + (readY ? w : 0) + (writeZ ? w : 0));
}

static double* part_tn(Ctx& c, int64_t q, int s) {
  return dbuf(c, "part_tn", tn_part_size(q, s));
}

static double* gram_buf(Ctx& c, int64_t q) {
  return dbuf(c, "gram", (size_t)nn_ctas(q, 1) * 32 * 32);
}

static double* scratch(Ctx& c, int64_t q) { return dbuf(c, "scratch", (size_t)q * 32); }

static int read_flags(Ctx& c) {
  TSVD_CUDA(cudaMemcpyAsync(c.hflags, c.dflags, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  TSVD_CUDA(cudaStreamSynchronize(c.st));
  return c.hflags[0] | c.hflags[1];
}

static void clear_flags(Ctx& c) {
  if (!c.deferred) TSVD_CUDA(cudaMemsetAsync(c.dflags, 0, 4 * sizeof(int), c.st));
}

// where this call's two breakdown flags go (see tsvd_ctx::deferred)
static int* ortho_flags(Ctx& c) {
  return c.deferred ? c.flag_log + 2 * c.flag_slot : c.dflags;
}

// immediate mode: sync and read the flags; deferred mode: never breaks down here
static int breakdown(Ctx& c) { return c.deferred ? 0 : read_flags(c); }

// Row-sharded reductions: every X^T Y or Gram computed on this
// rank's rows is a partial sum over the row partition; it is all-reduced
// before use so all ranks continue with identical small matrices.
// Single GPU: the finaliser sums the partials itself.  Row partition: sum
// here (same order), all-reduce, finalise the reduced W (np = 1).
static const double* reduce_gram(Ctx& c, const double* gram, int& np, int w, double* Wred) {
  if (!c.comm) return gram;
  gram_reduce(gram, np, w, Wred, c.st);
  allreduce_sum(c, Wred, (size_t)w * w);
  np = 1;
  return Wred;
}

// TRSM Q = Y L^{-T} (Alg. 4 S3/S6, Alg. 5 S5/S10) is applied as the product
// Y T with T = L^{-T} formed by the Cholesky finaliser (reading R30).
int cholqr2(Ctx& c, double* Y, int64_t q, int w, int64_t ld, double* R) {
  if (w > 32) throw Error{TSVD_EINVAL, "cholqr2: block wider than 32"};
  double* S = scratch(c, q);
  double* gram = gram_buf(c, q);
  double* Wred = dbuf(c, "Wred", 32 * 32);
  double* L1 = dbuf(c, "L1", 32 * 32);
  double* T1 = dbuf(c, "T1", 32 * 32);
  double* L2 = dbuf(c, "L2", 32 * 32);
  double* T2 = dbuf(c, "T2", 32 * 32);
  const int np = nn_ctas(q, w);
  clear_flags(c);
  {  // S1: W = Y^T Y
    Prof p(c, P_ROWT, nn_bytes(q, 0, w, true, false), 2.0 * q * w * w);
    gemm_nn(nullptr, 0, nullptr, 0, Y, ld, nullptr, nullptr, 0, q, 0, w, 0.0, 1.0, gram, c.st);
  }
  {
    Prof p(c, P_SMALL, 0, 0);
    int k = np;
    const double* W = reduce_gram(c, gram, k, w, Wred);
    chol_finalize(W, k, w, L1, T1, ortho_flags(c) + 0, c.st);                    // S2
  }
  {  // S3 + S4: S = Y L^{-T}, Wbar = S^T S
    Prof p(c, P_ROWT, nn_bytes(q, 0, w, true, true), 3.0 * q * w * w);
    gemm_nn(nullptr, 0, nullptr, 0, Y, ld, T1, S, w, q, 0, w, 0.0, 1.0, gram, c.st);
  }
  {
    Prof p(c, P_SMALL, 0, 0);
    int k = np;
    const double* W = reduce_gram(c, gram, k, w, Wred);
    chol2_finalize(W, k, w, L1, L2, T2, R, nullptr, nullptr, 0, ortho_flags(c) + 1, c.st);  // S5, S7
  }
  if (breakdown(c)) {
    Prof p(c, P_OTHER, 0, 0);
    cgs2(c, Y, q, 0, w, ld, nullptr, R);
    return 1;
  }
  {  // S6: Q = S Lbar^{-T}
    Prof p(c, P_ROWT, nn_bytes(q, 0, w, true, true), 1.0 * q * w * w);
    gemm_nn(nullptr, 0, nullptr, 0, S, w, T2, Y, ld, q, 0, w, 0.0, 1.0, nullptr, c.st);
  }
  return 0;
}

// BCGS-PIP+ (reading R34; oracle/core.py bcgs_pip2): two
// Pythagorean block CGS passes, each with ONE reduction.  Passes:
//   1 gemm_tn : C1 = [P Y]^T Y  (H1 = P^T Y, W1 = Y^T Y)      -> all-reduce C1
//     small   : M1 = W1 - H1^T H1, L1 = chol(M1), T1 = L1^{-T}, H1' = H1 T1
//   2 gemm_nn : Q1 = Y T1 - P H1'  (= (Y - P H1) L1^{-T}),  W2 = Q1^T Q1 (epilogue)
//   3 gemm_tn : H2 = P^T Q1                                     -> all-reduce [H2; W2]
//     small   : M2 = W2 - H2^T H2, L2, T2, H2' = H2 T2; R = L2^T L1^T; H = H1 + H2 L1^T
//   4 gemm_nn : Q = Q1 T2 - P H2'  (into Y's slot)
// Four basis reads like CGS-CQR2 but no basis-free TRSM / Gram passes (the
// TRSM rides in the NN epilogue through (Y - P H) T = Y T - P (H T)) and
// two reductions (multi-GPU: two all-reduces instead of four).
static int pip2(Ctx& c, double* basis, int64_t q, int s, int w, int64_t ld, double* H, double* R,
                bool need_h) {
  double* Y = basis + s;
  double* S = scratch(c, q);
  double* gram = gram_buf(c, q);
  double* part = part_tn(c, q, s + w);
  double* C1 = dbuf(c, "pip_C1", (size_t)(s + w) * w);
  double* C2 = dbuf(c, "pip_C2", (size_t)(s + w) * w);
  double* Hp = dbuf(c, "pip_Hp", (size_t)s * w);
  double* L1 = dbuf(c, "L1", 32 * 32);
  double* T1 = dbuf(c, "T1", 32 * 32);
  double* L2 = dbuf(c, "L2", 32 * 32);
  double* T2 = dbuf(c, "T2", 32 * 32);
  const int np = nn_ctas(q, w);
  clear_flags(c);
  const double fl = 2.0 * q * s * w;
  {
    Prof p(c, P_TN, tn_bytes(q, s + w, 0), 2.0 * q * (s + w) * w);
    gemm_tn(basis, ld, Y, ld, q, s + w, w, C1, w, part, c.st);                  // [H1; W1]
    allreduce_sum(c, C1, (size_t)(s + w) * w);
  }
  {  // M1 = W1 - H1^T H1, L1 = chol(M1), T1 = L1^{-T}, Hp = H1 T1
    Prof p(c, P_SMALL, 0, 0);
    pip_finalize(C1, s, w, L1, T1, Hp, ortho_flags(c) + 0, nullptr, nullptr, nullptr, nullptr,
                 c.st);
  }
  {
    Prof p(c, P_NN, nn_bytes(q, s, w, true, true), fl + 2.0 * q * w * w * 2);
    gemm_nn(basis, ld, Hp, w, Y, ld, T1, S, w, q, s, w, -1.0, 1.0, gram, c.st);  // Q1, W2
  }
  {
    Prof p(c, P_TN, tn_bytes(q, s, w), fl);
    gemm_tn(basis, ld, S, w, q, s, w, C2, w, part, c.st);                         // H2
  }
  {
    Prof p(c, P_SMALL, 0, 0);
    gram_reduce(gram, np, w, C2 + (size_t)s * w, c.st);                           // W2
    allreduce_sum(c, C2, (size_t)(s + w) * w);
    // L2, T2, Hp = H2 T2, R = L2^T L1^T, H = H1 + H2 L1^T
    pip_finalize(C2, s, w, L2, T2, Hp, ortho_flags(c) + 1, L1, R, C1,
                 (need_h && H) ? H : nullptr, c.st);
  }
  if (breakdown(c)) {
    Prof p(c, P_OTHER, 0, 0);
    cgs2(c, basis, q, s, w, ld, H, R);
    return 1;
  }
  {
    Prof p(c, P_NN, nn_bytes(q, s, w, true, true), fl + 2.0 * q * w * w);
    gemm_nn(basis, ld, Hp, w, S, w, T2, Y, ld, q, s, w, -1.0, 1.0, nullptr, c.st);  // Q
  }
  return 0;
}

int cgs_cqr2(Ctx& c, double* basis, int64_t q, int s, int w, int64_t ld, double* H,
             double* R, bool need_h) {
  if (s == 0) return cholqr2(c, basis, q, w, ld, R);
  if (w > 32) throw Error{TSVD_EINVAL, "cgs_cqr2: block wider than 32"};
  if (c.ortho == TSVD_ORTHO_BCGS_PIP2) return pip2(c, basis, q, s, w, ld, H, R, need_h);
  double* Y = basis + s;
  double* S = scratch(c, q);
  double* gram = gram_buf(c, q);
  double* part = part_tn(c, q, s);
  double* Wred = dbuf(c, "Wred", 32 * 32);
  double* L1 = dbuf(c, "L1", 32 * 32);
  double* T1 = dbuf(c, "T1", 32 * 32);
  double* L2 = dbuf(c, "L2", 32 * 32);
  double* T2 = dbuf(c, "T2", 32 * 32);
  double* Hbar = dbuf(c, "Hbar", (size_t)s * w);
  const int np = nn_ctas(q, w);
  clear_flags(c);
  const double fl = 2.0 * q * s * w;
  {
    Prof p(c, P_TN, tn_bytes(q, s, w), fl);
    gemm_tn(basis, ld, Y, ld, q, s, w, H, w, part, c.st);                             // S1
    allreduce_sum(c, H, (size_t)s * w);
  }
  {
    Prof p(c, P_NN, nn_bytes(q, s, w, true, true), fl + 2.0 * q * w * w);
    gemm_nn(basis, ld, H, w, Y, ld, nullptr, S, w, q, s, w, -1.0, 1.0, gram, c.st);   // S2,S3
  }
  {
    Prof p(c, P_SMALL, 0, 0);
    int k = np;
    const double* W = reduce_gram(c, gram, k, w, Wred);
    chol_finalize(W, k, w, L1, T1, ortho_flags(c) + 0, c.st);                         // S4
  }
  {
    Prof p(c, P_ROWT, nn_bytes(q, 0, w, true, true), 1.0 * q * w * w);
    gemm_nn(nullptr, 0, nullptr, 0, S, w, T1, S, w, q, 0, w, 0.0, 1.0, nullptr, c.st);  // S5
  }
  {
    Prof p(c, P_TN, tn_bytes(q, s, w), fl);
    gemm_tn(basis, ld, S, w, q, s, w, Hbar, w, part, c.st);                           // S6
    allreduce_sum(c, Hbar, (size_t)s * w);
  }
  {
    Prof p(c, P_NN, nn_bytes(q, s, w, true, true), fl + 2.0 * q * w * w);
    gemm_nn(basis, ld, Hbar, w, S, w, nullptr, S, w, q, s, w, -1.0, 1.0, gram, c.st);  // S7,S8
  }
  {
    Prof p(c, P_SMALL, 0, 0);
    int k = np;
    const double* W = reduce_gram(c, gram, k, w, Wred);
    chol2_finalize(W, k, w, L1, L2, T2, R, need_h ? H : nullptr, Hbar, s, ortho_flags(c) + 1,
                   c.st);                                                             // S9,S11,S12
  }
  if (breakdown(c)) {
    Prof p(c, P_OTHER, 0, 0);
    cgs2(c, basis, q, s, w, ld, H, R);
    return 1;
  }
  {
    Prof p(c, P_ROWT, nn_bytes(q, 0, w, true, true), 1.0 * q * w * w);
    gemm_nn(nullptr, 0, nullptr, 0, S, w, T2, Y, ld, q, 0, w, 0.0, 1.0, nullptr, c.st);  // S10
  }
  return 0;
}

// Column-wise CGS with reorthogonalisation against [P, Q_<j] (
// reading R16).  Y = columns [s, s+w) of basis is processed in place; H (s x w)
// and R (w x w) receive the coefficients.  Replacement columns are rows
// [cur_row0, cur_row0 + q) of a cur_qtot-row Philox column, so every rank of a
// row partition draws its own rows of the same global vector.
void cgs2(Ctx& c, double* basis, int64_t q, int s, int w, int64_t ld, double* H, double* R) {
  const double tau = 1e-13;
  double* S = dbuf(c, "cgs2_col", (size_t)q);
  double* gram = gram_buf(c, q);
  const int np = nn_ctas(q, 1);
  double* c1 = dbuf(c, "cgs2_c1", (size_t)(s + w));
  double* c2 = dbuf(c, "cgs2_c2", (size_t)(s + w));
  double* coef = dbuf(c, "cgs2_coef", (size_t)(s + w));
  double* sc = dbuf(c, "cgs2_sc", 8);  // [0] |y_orig|^2, [1] |y''|^2, [2] nrm
  double* part = part_tn(c, q, s + w);
  int* dep = c.dflags + 2;
  const int64_t row0 = c.cur_row0, qtot = c.cur_qtot > 0 ? c.cur_qtot : q;
  auto gram1 = [&](double* out) {
    reduce_partials(gram, np, 1, out, c.st);
    allreduce_sum(c, out, 1);
  };
  auto proj = [&](const double* x, int64_t ldx2, double* cc, int nb) {
    gemm_tn(basis, ld, x, ldx2, q, nb, 1, cc, 1, part, c.st);
    allreduce_sum(c, cc, (size_t)nb);
  };
  ++c.breakdowns;
  fill_zero(R, (int64_t)w * w, c.st);
  for (int j = 0; j < w; ++j) {
    const int nb = s + j;
    double* col = basis + s + j;
    // ||y_orig||^2
    gemm_nn(nullptr, 0, nullptr, 0, col, ld, nullptr, nullptr, 0, q, 0, 1, 0.0, 1.0, gram, c.st);
    gram1(sc + 0);
    if (nb > 0) {
      proj(col, ld, c1, nb);
      gemm_nn(basis, ld, c1, 1, col, ld, nullptr, S, 1, q, nb, 1, -1.0, 1.0, nullptr, c.st);
      proj(S, 1, c2, nb);
      gemm_nn(basis, ld, c2, 1, S, 1, nullptr, S, 1, q, nb, 1, -1.0, 1.0, gram, c.st);
    } else {
      gemm_nn(nullptr, 0, nullptr, 0, col, ld, nullptr, S, 1, q, 0, 1, 0.0, 1.0, gram, c.st);
    }
    gram1(sc + 1);
    cgs2_col_finalize(c1, c2, nb, sc + 1, sc + 0, tau, coef, sc + 2, dep, c.st);
    int hdep = 0;
    TSVD_CUDA(cudaMemcpyAsync(&hdep, dep, sizeof(int), cudaMemcpyDeviceToHost, c.st));
    TSVD_CUDA(cudaStreamSynchronize(c.st));
    if (hdep) {
      // replacement column: next Philox draw, orthogonalised twice
      launch_philox_normal(S, q, 1, 1, c.seed, c.draw_next++, row0, qtot, c.st);
      for (int it = 0; it < 2 && nb > 0; ++it) {
        proj(S, 1, c2, nb);
        gemm_nn(basis, ld, c2, 1, S, 1, nullptr, S, 1, q, nb, 1, -1.0, 1.0, nullptr, c.st);
      }
      gemm_nn(nullptr, 0, nullptr, 0, S, 1, nullptr, nullptr, 0, q, 0, 1, 0.0, 1.0, gram, c.st);
      gram1(sc + 1);
      cgs2_col_finalize(c1, c1, 0, sc + 1, sc + 1, 0.0, coef + nb, sc + 2, dep, c.st);
      ++c.replaced;
    } else {
      TSVD_CUDA(cudaMemcpyAsync(R + (int64_t)j * w + j, sc + 2, sizeof(double),
                                cudaMemcpyDeviceToDevice, c.st));
    }
    // Q_j = S / nrm
    copy_block(S, 1, col, ld, q, 1, false, c.st);
    scale_column(col, q, ld, sc + 2, c.st);
    if (s > 0 && H) copy_block(coef, 1, H + j, w, s, 1, false, c.st);
    if (j > 0) copy_block(coef + s, 1, R + j, w, j, 1, false, c.st);
  }
}

// LancSVD's block orthogonalisation for any block width b (b >= 1):
// the columns [s, s + b) of `basis` against [0, s), R (b x b, ld b) with
// Y = P H + Q R (H discarded, reading R17).  b <= 32: one CholQR2 (s = 0) or
// CGS-CQR2 call.  Wider blocks go in 32-column panels exactly like Alg. 3
// (CGS-QR): panel j against P and the earlier panels, R's column block j =
// [the earlier panels' rows of H_j; R_jj].  The QR with positive diagonal is
// unique, so this is the oracle's b-wide CholQR2 / CGS-CQR2 up to rounding.
int block_orth(Ctx& c, double* basis, int64_t q, int s, int b, int64_t ld, double* R) {
  if (b <= 32) {
    if (s == 0) return cholqr2(c, basis, q, b, ld, R);
    double* H = dbuf(c, "H", (size_t)s * 32);
    return cgs_cqr2(c, basis, q, s, b, ld, H, R, false);
  }
  int bd = 0;
  fill_zero(R, (int64_t)b * b, c.st);
  double* Hj = dbuf(c, "borth_H", (size_t)(s + b) * 32);
  double* Rj = dbuf(c, "borth_R", 32 * 32);
  for (int j0 = 0; j0 < b; j0 += 32) {
    const int w = std::min(32, b - j0);
    if (s + j0 == 0) {
      bd += cholqr2(c, basis, q, w, ld, Rj);
    } else {
      bd += cgs_cqr2(c, basis, q, s + j0, w, ld, Hj, Rj, true);
      if (j0 > 0) copy_block(Hj + (size_t)s * w, w, R + j0, b, j0, w, false, c.st);
    }
    copy_block(Rj, w, R + (int64_t)j0 * b + j0, b, w, w, false, c.st);
  }
  return bd;
}

int cgs_qr(Ctx& c, double* Y, int64_t q, int l, int64_t ld, int bq, double* R) {
  int bd = 0;
  fill_zero(R, (int64_t)l * l, c.st);
  double* Hj = dbuf(c, "cgsqr_H", (size_t)l * 32);
  double* Rj = dbuf(c, "cgsqr_R", 32 * 32);
  for (int s0 = 0; s0 < l; s0 += bq) {
    const int w = std::min(bq, l - s0);
    if (s0 == 0) {
      bd += cholqr2(c, Y, q, w, ld, Rj);                       // Alg. 3 S1
    } else {
      bd += cgs_cqr2(c, Y, q, s0, w, ld, Hj, Rj);              // Alg. 3 S2
      copy_block(Hj, w, R + s0, l, s0, w, false, c.st);        // [H_j; R_j]
    }
    copy_block(Rj, w, R + (int64_t)s0 * l + s0, l, w, w, false, c.st);
  }
  return bd;
}

// Products with A on this rank's rows (Alg. 1 S1/S3, Alg. 2 S2/S4).
//  trans = 0: Y (m_loc x w) = A_g X, X = this rank's n-shard (n_loc x w);
//             multi-GPU: the n-shards are all-gathered into the full X first.
//  trans = 1: Y (n_loc x w) = (A^T X)[n-shard], X = this rank's rows (m_loc x w);
//             multi-GPU: the full-n partial A_g^T X is reduce-scattered.
static void apply_local(Ctx& c, bool trans, const double* X, int64_t ldx, double* Y,
                        int64_t ldy, int w) {
  const double rows = trans ? (double)c.ng : (double)c.m, cols = trans ? (double)c.m : (double)c.ng;
  const double bytes = c.dense ? 8.0 * ((double)c.m * c.ng + w * (rows + cols))
                               : 12.0 * c.A.nnz + 8.0 * (rows + 1) + 8.0 * w * (rows + cols);
  const double flops = c.dense ? 2.0 * c.m * c.ng * w : 2.0 * c.A.nnz * w;
  Prof p(c, trans ? P_APPLY_AT : P_APPLY_A, bytes, flops);
  if (c.dense) {
    if (!trans) {
      // split-K scratch for the few-row-tile dense product (ts.cu pick_split)
      const bool few_tiles = c.m < (int64_t)128 * 8 * 148;
      const size_t cap = few_tiles ? (size_t)8 * c.m * std::min(w, 64) : 0;
      double* part = few_tiles ? dbuf(c, "nn_split", cap) : nullptr;
      gemm_nn(c.Ad, c.lda, X, ldx, nullptr, 0, nullptr, Y, ldy, c.m, (int)c.ng, w, 1.0, 0.0,
              nullptr, c.st, part, cap);
    }
    else
      gemm_tn(c.Ad, c.lda, X, ldx, c.m, (int)c.ng, w, Y, ldy, part_tn(c, c.m, (int)c.ng), c.st);
  } else {
    const Csr& A = trans ? c.AT : c.A;
    double* part = dbuf(c, trans ? "spmm_part_t" : "spmm_part",
                        (size_t)std::max<int64_t>(1, A.nslots) * 64);
    launch_spmm_wide(A, X, ldx, Y, ldy, w, part, c.st);
  }
}

void apply(Ctx& c, bool trans, const double* X, int64_t ldx, double* Y, int64_t ldy, int w) {
  if (!c.comm) {
    apply_local(c, trans, X, ldx, Y, ldy, w);
    return;
  }
  const int64_t npad = c.nsh * c.world;
  double* full = dbuf(c, "dist_full", (size_t)npad * w);
  double* shard = dbuf(c, "dist_shard", (size_t)c.nsh * w);
  if (!trans) {
    // all-gather the n-shards of X (zero-padded to nsh rows) into full n
    fill_zero(shard, c.nsh * w, c.st);
    copy_block(X, ldx, shard, w, c.n, w, false, c.st);
    {
      Prof p(c, P_OTHER, 8.0 * npad * w, 0);
      all_gather(c, shard, full, (size_t)c.nsh * w);
    }
    apply_local(c, false, full, w, Y, ldy, w);
  } else if (!c.ATp.empty() && !c.dense) {
    // pipelined reduce-scatter: the partial A_g^T X is formed
    // one n-shard at a time from the row pieces of CSR(A_g^T); as soon as
    // shard p is written, its reduction to rank p (ncclReduce, in shard
    // order on every rank) starts on the communication stream while the
    // compute stream multiplies shard p + 1
    if (!c.comm_st) {
      TSVD_CUDA(cudaStreamCreateWithFlags(&c.comm_st, cudaStreamNonBlocking));
      c.comm_ev.resize(c.world + 1);
      for (auto& e : c.comm_ev) TSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int64_t tail = npad - c.ng;  // padding rows of the last shard stay zero
    if (tail > 0) fill_zero(full + (size_t)c.ng * w, tail * w, c.st);
    Prof p(c, P_APPLY_AT, 12.0 * c.AT.nnz + 8.0 * (c.ng + 1) + 8.0 * w * (c.ng + c.m),
           2.0 * c.AT.nnz * w);
    int64_t slots = std::max<int64_t>(1, c.AT.nslots);
    for (const Csr& P : c.ATp) slots = std::max(slots, P.nslots);
    double* part = dbuf(c, "spmm_part_t", (size_t)slots * 64);
    for (int g = 0; g < c.world; ++g) {
      const Csr& P = c.ATp[g];
      double* out = full + (size_t)g * c.nsh * w;
      if (P.rows > 0) launch_spmm_wide(P, X, ldx, out, w, w, part, c.st);
      TSVD_CUDA(cudaEventRecord(c.comm_ev[g], c.st));
      TSVD_CUDA(cudaStreamWaitEvent(c.comm_st, c.comm_ev[g], 0));
      reduce_sum_to(c, out, shard, (size_t)c.nsh * w, g, c.comm_st);
    }
    TSVD_CUDA(cudaEventRecord(c.comm_ev[c.world], c.comm_st));
    TSVD_CUDA(cudaStreamWaitEvent(c.st, c.comm_ev[c.world], 0));
    copy_block(shard, w, Y, ldy, c.n, w, false, c.st);
  } else {
    fill_zero(full, npad * w, c.st);
    apply_local(c, true, X, ldx, full, w, w);
    {
      Prof p(c, P_OTHER, 8.0 * npad * w, 0);
      reduce_scatter_sum(c, full, shard, (size_t)c.nsh * w);
    }
    copy_block(shard, w, Y, ldy, c.n, w, false, c.st);
  }
}

}  // namespace tsvd
