// Solver drivers: LancSVD (Alg. 2) and RandSVD (Alg. 1,
// P:66-92).  Host loops that enqueue the device building blocks on the
// handle's stream; the host reads one flag per orthogonalisation (breakdown,
// P:275) and rho/sigma once per restart cycle.
//
// Layout in HBM: the Lanczos bases are row-major
// panels Pbar (m x (d+b)) and P (n x d); block i lives in columns
// [i b, (i+1) b), so one row of [P_{i-1} | Q_i] is one contiguous segment and
// the orthogonalisation kernels read each basis row once per pass.  Column
// block k of Pbar holds Qbar_{k+1} (reading R18), later reused as the slot
// for the restart product.
#include <algorithm>
#include <cmath>

#include "ctx.h"

namespace tsvd {

bool g_svd_overlap = getenv("TSVD_SVD_OVERLAP") ? atoi(getenv("TSVD_SVD_OVERLAP")) != 0 : true;
constexpr int kSvdHogSmem = 160 * 1024;
constexpr int kSvdOverlapRows = 4000;

static void upload_start(Ctx& c, double* dst, int64_t rows, int cols, int64_t ld) {
  TSVD_CUDA(cudaMemcpy2DAsync(dst, ld * sizeof(double), c.start.data(), cols * sizeof(double),
                              cols * sizeof(double), rows, cudaMemcpyHostToDevice, c.st));
}

// sign of the largest-|.| entry of each column of the (row-sharded) V (R28)
static double* signs_of(Ctx& c, const double* V, int64_t n, int64_t ldv, int r) {
  double* work = dbuf(c, "sign_work", col_signs_work(r, c.world));
  double* sgn = dbuf(c, "sign", (size_t)r);
  double* loc = col_signs_local(V, n, ldv, r, c.n0, work, c.st);
  if (c.comm) {
    double* all = dbuf(c, "sign_all", (size_t)3 * r * c.world);
    all_gather(c, loc, all, (size_t)3 * r);
    col_signs_final(all, c.world, r, sgn, c.st);
  } else {
    col_signs_final(loc, 1, r, sgn, c.st);
  }
  return sgn;
}

// tsvd_set_output_mode: form U_r, V_r in place over the bases when separate
// m x r and n x r buffers do not fit in the free device memory (C5 on one GPU).
static bool outputs_in_place(Ctx& c, int r, const char* nu = "res_U", const char* nv = "res_V") {
  if (c.out_mode == TSVD_OUT_INPLACE) return true;
  if (c.out_mode == TSVD_OUT_SEPARATE) return false;
  size_t have = 0;
  for (const char* nm : {nu, nv}) {
    auto it = c.bufs.find(nm);
    if (it != c.bufs.end()) have += it->second.second;
  }
  const size_t need = (size_t)(c.m + c.n) * r * sizeof(double);
  if (need <= have) return false;
  size_t fr = 0, tot = 0;
  TSVD_CUDA(cudaMemGetInfo(&fr, &tot));
  int dev = 0;
  cudaMemPool_t pool;
  size_t pool_free = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t res = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
        res > used)
      pool_free = (size_t)(res - used);
  }
  cudaGetLastError();
  const size_t margin = (size_t)2 << 30;
  return need - have + margin > fr + pool_free;
}

// Output product Z = X[:, :s] H[:, :r] (Eq. 12; Alg. 1 S6/S7), row-local.
// Separate: into the named result buffer.  In place: over X's first r
// columns, in row chunks staged through the pass scratch buffer (a chunk's
// rows are read completely by the product before the copy overwrites them).
static double* out_product(Ctx& c, const char* name, double* X, int64_t ldx, int64_t rows,
                           int s, const double* H, int64_t ldh, int r, bool inplace,
                           int64_t* ld) {
  if (!inplace) {
    double* Z = dbuf(c, name, (size_t)rows * r);
    gemm_nn(X, ldx, H, ldh, nullptr, 0, nullptr, Z, r, rows, s, r, 1.0, 0.0, nullptr, c.st);
    *ld = r;
    return Z;
  }
  if (gemm_nn_out_inplace(X, ldx, H, ldh, rows, s, r, c.st)) {  // one pass, no scratch
    *ld = ldx;
    return X;
  }
  const size_t cap = (size_t)std::max(c.m, c.n) * 32;  // pre-sized by the solvers
  double* stage = dbuf(c, "scratch", cap);
  const int64_t chunk = std::max<int64_t>(1, (int64_t)(cap / r));
  for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
    const int64_t rc = std::min(chunk, rows - r0);
    gemm_nn(X + r0 * ldx, ldx, H, ldh, nullptr, 0, nullptr, stage, r, rc, s, r, 1.0, 0.0,
            nullptr, c.st);
    copy_block(stage, r, X + r0 * ldx, ldx, rc, r, false, c.st);
  }
  *ld = ldx;
  return X;
}

struct EventTimer {
  cudaEvent_t a, b;
  cudaStream_t st;
  explicit EventTimer(cudaStream_t s) : st(s) {
    TSVD_CUDA(cudaEventCreate(&a));
    TSVD_CUDA(cudaEventCreate(&b));
    TSVD_CUDA(cudaEventRecord(a, st));
  }
  double stop() {
    TSVD_CUDA(cudaEventRecord(b, st));
    TSVD_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    TSVD_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// Deferred breakdown checks (tsvd_ctx::deferred) must never outlive the
// solve that set them: an exception leaving the block-step loop (ENOMEM, a
// CUDA or NCCL error) would otherwise leave a later solve on this handle
// skipping its breakdown test and writing into a stale flag log.
struct DeferredGuard {
  Ctx& c;
  explicit DeferredGuard(Ctx& c_) : c(c_) { reset(); }
  ~DeferredGuard() { reset(); }
  void reset() {
    c.deferred = false;
    c.flag_log = nullptr;
    c.flag_slot = 0;
  }
};

// Sweep count of the SVD just enqueued, read with the cycle's other scalars.
struct SvdWatch {
  int max_sweeps = 0, unconverged = 0;
  void add(unsigned sweeps) {
    max_sweeps = std::max(max_sweeps, (int)sweeps);
    if ((int)sweeps >= small_svd_max_sweeps()) ++unconverged;
  }
};

tsvd_status lanczos_solve(Ctx& c, int r, int b, double tol, int maxit) {
  const int64_t m = c.m, n = c.n;  // this rank's rows (single GPU: all)
  DeferredGuard guard(c);
  if (r < 1 || b < 1 || !(tol > 0.0) || maxit < 1) return TSVD_EINVAL;
  if (r > c.ng) return TSVD_ESHAPE;
  int d = c.krylov_d;
  if (d == 0) {
    d = std::max(4 * r, 2 * b);
    d = (int)std::min<int64_t>(d, c.ng);
    d = std::min(d, kSmallSvdMaxD);
    d -= d % b;
  }
  if (d % b != 0 || d < r || d > c.ng || d < b || d > kSmallSvdMaxD) return TSVD_ESHAPE;
  if (!c.start.empty() && (c.start_rows != m || c.start_cols != b)) return TSVD_ESHAPE;
  const int keep = c.thick_keep;  // N1 thick restart (0: Alg. 2 S7)
  if (keep && (keep % b != 0 || keep < r || keep >= d)) return TSVD_ESHAPE;
  const int k = d / b;
  const int64_t ldb = d + b, ldp = d;
  c.have = false;
  c.breakdowns = 0;
  c.replaced = 0;
  c.draw_next = 1;
  const int64_t launches0 = g_launches.load();
  EventTimer timer(c.st);

  double* Pb = dbuf(c, "Pbar", (size_t)m * ldb);
  double* P = dbuf(c, "P", (size_t)n * ldp);
  double* B = dbuf(c, "B", (size_t)d * d);
  double* Ub = dbuf(c, "Ub", (size_t)d * d);
  double* Vb = dbuf(c, "Vb", (size_t)d * d);
  double* Sg = dbuf(c, "Sg", (size_t)d);
  // a previous solve that ended in an error may have left its forked SVD
  // running on buffers this one reuses (normally the side stream is idle)
  if (c.svd_st) TSVD_CUDA(cudaStreamSynchronize(c.svd_st));
  double* jw = dbuf(c, "jacobi_work", small_svd_work(d));
  // the SVD's own TN scratch: with the overlap below it runs beside the last
  // m-side orthogonalisation, which uses part_tn
  double* part_svd = dbuf(c, "part_svd", tn_part_size(d, d));
  (void)dbuf(c, "H", (size_t)d * 32);
  const size_t rb = (size_t)std::max(32, b);
  double* R = dbuf(c, "R", rb * rb);
  double* Rb = dbuf(c, "Rb", rb * rb);
  double* rho = dbuf(c, "rho", (size_t)d);
  // pre-size the pass workspaces for the largest q and s of this solve
  (void)dbuf(c, "scratch", (size_t)std::max(m, n) * 32);
  (void)dbuf(c, "gram", (size_t)nn_ctas(std::max(m, n), 1) * 32 * 32);
  (void)dbuf(c, "Hbar", (size_t)(d + b) * 32);
  (void)dbuf(c, "part_tn", std::max(tn_part_size(m, d + b), tn_part_size(n, d)));

  // S1: random orthonormal Qbar_1 (m x b); rows [m0, m0+m) of the global block
  auto m_side = [&]() { c.cur_row0 = c.m0; c.cur_qtot = c.mg; };
  auto n_side = [&]() { c.cur_row0 = c.n0; c.cur_qtot = c.ng; };
  if (!c.start.empty())
    upload_start(c, Pb, m, b, ldb);
  else
    launch_philox_normal(Pb, m, b, ldb, c.seed, 0, c.m0, c.mg, c.st);
  m_side();
  block_orth(c, Pb, m, 0, b, ldb, R);

  std::vector<double> hrho(r), hs(1);
  unsigned* hsw = reinterpret_cast<unsigned*>(c.hflags + 4);  // pinned word
  SvdWatch svdw;
  int cycle = 0, nconv = 0;
  bool conv = false;
  double rho_max = 0.0;
  int* flog = (int*)buf(c, "flag_log", sizeof(int) * 4 * (size_t)k);
  std::vector<int> hlog(4 * (size_t)k);
  fill_zero(B, (int64_t)d * d, c.st);
  int s0 = 0;  // columns carried over by a thick restart (block steps start there)
  int kc = 0;   // block steps of the current cycle
  // Alg. 2 S2-S5 for block step i of the current cycle (both sides, or only
  // the m side when a replay starts at the m-side slot of step i)
  auto block_step = [&](int i, bool n_part = true) {
    const int lo = s0 + i * b;
    if (n_part) {
      apply(c, true, Pb + lo, ldb, P + lo, ldp, b);                  // S2: A^T Qbar_i
      n_side();
      c.flag_slot = 2 * i;
      block_orth(c, P, n, lo, b, ldp, R);                            // S3a / S3b (H unused, R17)
      copy_block(R, b, B + (int64_t)lo * d + lo, d, b, b, true, c.st);  // L_i = R^T
    }
    apply(c, false, P + lo, ldp, Pb + lo + b, ldb, b);               // S4: A Q_i
    m_side();
    c.flag_slot = 2 * i + 1;
    block_orth(c, Pb, m, lo + b, b, ldb, Rb);                        // S5 (H unused, R17)
    if (i < kc - 1)
      copy_block(Rb, b, B + (int64_t)(lo + b) * d + lo, d, b, b, false, c.st);  // Rbar_i
  };
  for (cycle = 1; cycle <= maxit; ++cycle) {
    kc = (d - s0) / b;
    // Block steps, first with deferred breakdown checks (no host sync per
    // orthogonalisation); if the log shows a breakdown in call `slot`
    // (2i: n side of step i, 2i+1: m side) the steps are replayed from there
    // with immediate checks and the CGS2 fallback.
    TSVD_CUDA(cudaMemsetAsync(flog, 0, sizeof(int) * 4 * (size_t)k, c.st));
    c.flag_log = flog;
    c.deferred = true;
    int from_slot = 0;
    // The deferred pass has no host synchronisation, so on a single GPU it is
    // replayed as a CUDA graph once the same cycle shape was seen before (the
    // first run allocates every workspace; the capture then only records).
    CycleGraph& cg = c.cyc_graph;
    const void* ptrs[4] = {Pb, P, B, flog};
    const bool graph_ok = c.graphs && !c.comm;
    bool same = graph_ok && cg.m == m && cg.n == n && cg.d == d && cg.b == b && cg.s0 == s0 &&
                cg.kc == kc && cg.ortho == c.ortho && cg.prof == c.prof_mask &&
                cg.bufgen == c.bufgen && std::equal(ptrs, ptrs + 4, cg.ptrs);
    if (graph_ok && !same) {
      cycle_graph_reset(c);
      cg.m = m, cg.n = n, cg.d = d, cg.b = b, cg.s0 = s0, cg.kc = kc, cg.ortho = c.ortho;
      cg.prof = c.prof_mask;
      cg.bufgen = c.bufgen;
      std::copy(ptrs, ptrs + 4, cg.ptrs);
    }
    bool graph_ran = false;
    if (same && !cg.exec && cg.seen >= 1) {
      // capture the block steps exactly as the eager loop below enqueues them
      const size_t prof0 = c.prof_open.size();
      const int64_t l0 = g_launches.load();
      c.capturing = true;
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal);
      if (ce == cudaSuccess) {
        try {
          for (int i = 0; i < kc; ++i) block_step(i);
        } catch (...) {
          c.capturing = false;
          cudaStreamEndCapture(c.st, &graph);
          if (graph) cudaGraphDestroy(graph);
          cudaGetLastError();
          throw;
        }
        ce = cudaStreamEndCapture(c.st, &graph);
      }
      c.capturing = false;
      if (ce == cudaSuccess) ce = cudaGraphInstantiate(&cg.exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      cg.launches = g_launches.load() - l0;
      g_launches.fetch_sub(cg.launches);  // nothing ran yet
      for (size_t j = prof0; j < c.prof_open.size(); ++j) {
        c.prof_open[j].graph_owned = true;
        cg.prof_recs.push_back(c.prof_open[j]);
      }
      c.prof_open.resize(prof0);
      if (ce != cudaSuccess) {  // not capturable here: stay eager
        cudaGetLastError();
        cycle_graph_reset(c);
        c.graphs = false;
      }
    }
    if (same && cg.exec) {
      TSVD_CUDA(cudaGraphLaunch(cg.exec, c.st));
      g_launches.fetch_add(cg.launches + 1);
      c.prof_open.insert(c.prof_open.end(), cg.prof_recs.begin(), cg.prof_recs.end());
      graph_ran = true;
    } else if (graph_ok) {
      ++cg.seen;
    }
    // B_k is complete once the n side of the last block step has written
    // L_k (the m side only adds Rbar_k, which goes to Rb for rho, not into
    // B), so on one GPU the Jacobi SVD of B_k -- latency-bound on a few
    // dozen SMs -- runs on a side stream beside that last m-side product and
    // orthogonalisation (TSVD_SVD_OVERLAP=0: after them).  A breakdown replay
    // rewrites B, so it waits for the early SVD and the SVD runs again.
    const int nv = std::min(d, std::max(r, keep));
    bool svd_early = false;
    auto fork_svd = [&]() {
      if (!c.svd_st) {
        TSVD_CUDA(cudaStreamCreateWithFlags(&c.svd_st, cudaStreamNonBlocking));
        TSVD_CUDA(cudaEventCreateWithFlags(&c.svd_fork, cudaEventDisableTiming));
        TSVD_CUDA(cudaEventCreateWithFlags(&c.svd_join, cudaEventDisableTiming));
      }
      TSVD_CUDA(cudaEventRecord(c.svd_fork, c.st));
      TSVD_CUDA(cudaStreamWaitEvent(c.svd_st, c.svd_fork, 0));
      cudaStream_t main_st = c.st;
      c.st = c.svd_st;  // the phase events of this SVD go on its stream
      try {
        Prof p(c, P_SVD, 16.0 * d * d, 0);
        small_svd_top(B, d, nv, Ub, Sg, Vb, jw, part_svd, c.svd_st, kSvdHogSmem);
      } catch (...) {
        c.st = main_st;
        throw;
      }
      c.st = main_st;
      TSVD_CUDA(cudaEventRecord(c.svd_join, c.svd_st));
      svd_early = true;
    };
    // only where the SVD outlasts that m-side step: the streaming passes then
    // run on the SMs the Jacobi leaves free (its CTAs reserve shared memory,
    // kSvdHogSmem, so no pass CTA shares an SM with them: sharing slowed the
    // latency-bound Jacobi 1.3-2.5x).  m < kSvdOverlapRows d: C2 (m/d = 2604)
    // and the dense C4 (57) overlap, C3 (6250) and C5 do not -- there the
    // m-side orthogonalisation on the remaining SMs would outlast the SVD.
    const bool overlap_ok = g_svd_overlap && !c.comm && !graph_ran &&
                            (c.dense || m < (int64_t)kSvdOverlapRows * d);
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = (pass == 0 && graph_ran) ? kc : from_slot / 2; i < kc; ++i) {
        const bool n_part = !(i == from_slot / 2 && (from_slot & 1));
        if (pass == 0 && overlap_ok && i == kc - 1 && n_part) {
          const int lo = s0 + i * b;
          apply(c, true, Pb + lo, ldb, P + lo, ldp, b);
          n_side();
          c.flag_slot = 2 * i;
          block_orth(c, P, n, lo, b, ldp, R);
          copy_block(R, b, B + (int64_t)lo * d + lo, d, b, b, true, c.st);
          fork_svd();
          c.prof_override = P_BESIDE_SVD;
          try {
            block_step(i, false);
          } catch (...) {
            c.prof_override = -1;
            throw;
          }
          c.prof_override = -1;
        } else {
          block_step(i, n_part);
        }
      }
      if (svd_early) {  // joined before anything else reads or rewrites B, Ub, Sg, Vb
        TSVD_CUDA(cudaStreamWaitEvent(c.st, c.svd_join, 0));
      }
      if (!c.deferred) break;
      TSVD_CUDA(cudaMemcpyAsync(hlog.data(), flog, sizeof(int) * 4 * (size_t)k,
                                cudaMemcpyDeviceToHost, c.st));
      TSVD_CUDA(cudaStreamSynchronize(c.st));
      if (graph_ran) prof_harvest(c);  // the graph's events are re-recorded by the next replay
      c.deferred = false;
      int bad = -1;
      for (int sl = 0; sl < 2 * kc && bad < 0; ++sl)
        if (hlog[2 * sl] || hlog[2 * sl + 1]) bad = sl;
      if (bad < 0) break;
      from_slot = bad;
      svd_early = false;  // the replay changes B: the SVD runs again below
    }
    c.deferred = false;
    // B_k = Ub S Vb^T.  Only Vbar[:, :max(r, l)] is ever read (rho, outputs,
    // thick restart), so the sweeps skip V and those columns are formed as
    // B^T ubar_i / sigma_i (small_svd_top); if sigma_max(r,l) < 1e-3 sigma_1 the
    // full Jacobi with rotated V runs instead (host-checked with rho below).
    for (int full = 0; full < 2; ++full) {
      if (!(full == 0 && svd_early)) {
        Prof p(c, P_SVD, 16.0 * d * d, 0);
        if (full)
          small_svd(B, d, Ub, Sg, Vb, jw, c.st);
        else
          small_svd_top(B, d, nv, Ub, Sg, Vb, jw, part_svd, c.st);
      }
      {
        Prof p(c, P_OTHER, 0, 0);
        lanczos_rho(Rb, b, Vb, d, Sg, r, rho, c.st);
      }
      TSVD_CUDA(cudaMemcpyAsync(hrho.data(), rho, r * sizeof(double), cudaMemcpyDeviceToHost, c.st));
      TSVD_CUDA(cudaMemcpyAsync(hs.data(), Sg, sizeof(double), cudaMemcpyDeviceToHost, c.st));
      TSVD_CUDA(cudaMemcpyAsync(hsw, small_svd_sweeps_dev(jw, d), sizeof(unsigned),
                                cudaMemcpyDeviceToHost, c.st));
      if (!full)
        TSVD_CUDA(cudaMemcpyAsync(hsw + 1, small_svd_top_ok_dev(jw, d), sizeof(unsigned),
                                  cudaMemcpyDeviceToHost, c.st));
      TSVD_CUDA(cudaStreamSynchronize(c.st));
      svdw.add(*hsw);
      if (full || hsw[1]) break;
    }
    nconv = 0;
    rho_max = 0.0;
    for (int i = 0; i < r; ++i) {
      if (hrho[i] <= tol) ++nconv;
      rho_max = std::max(rho_max, hrho[i]);
    }
    conv = (nconv == r);
    if (conv || cycle == maxit) break;
    if (keep) {
      // N1 thick restart (oracle/lancsvd.py header): Pbar' = Pbar_k Ubar[:, :l],
      // P' = P_k Vbar[:, :l] (computed into scratch panels, then copied over
      // the bases' first l columns), Qbar_{k+1} moved behind them, and the
      // next B' starts as [Sigma_l; S] with S = Rbar_k Vbar[d-b:d, :l].
      {
        Prof p(c, P_RESTART, 8.0 * (m + n) * (d + 3.0 * keep) + 16.0 * m * b,
               2.0 * (m + n) * d * keep);
        if (outputs_in_place(c, keep, "thick_Pb", "thick_P")) {
          // no room for m x l / n x l panels (C5 on one GPU): the row-local
          // products overwrite the bases' first l columns through the pass
          // scratch, chunk by chunk (out_product, as for the outputs)
          int64_t ld_unused = 0;
          out_product(c, "thick_Pb", Pb, ldb, m, d, Ub, d, keep, true, &ld_unused);
          out_product(c, "thick_P", P, ldp, n, d, Vb, d, keep, true, &ld_unused);
        } else {
          double* tPb = dbuf(c, "thick_Pb", (size_t)m * keep);
          double* tP = dbuf(c, "thick_P", (size_t)n * keep);
          gemm_nn(Pb, ldb, Ub, d, nullptr, 0, nullptr, tPb, keep, m, d, keep, 1.0, 0.0, nullptr,
                  c.st);
          gemm_nn(P, ldp, Vb, d, nullptr, 0, nullptr, tP, keep, n, d, keep, 1.0, 0.0, nullptr,
                  c.st);
          copy_block(tPb, keep, Pb, ldb, m, keep, false, c.st);
          copy_block(tP, keep, P, ldp, n, keep, false, c.st);
        }
        copy_block(Pb + d, ldb, Pb + keep, ldb, m, b, false, c.st);
      }
      fill_zero(B, (int64_t)d * d, c.st);
      thick_arrow(Rb, b, Vb, d, Sg, keep, B, c.st);
      s0 = keep;
      continue;
    }
    fill_zero(B, (int64_t)d * d, c.st);
    // S7: Qbar_1 = Pbar_k Ubar_1 (first b left Ritz vectors, reading R19),
    // re-orthonormalised (reading R11); computed into the spare slot.
    {
      Prof p(c, P_RESTART, 8.0 * m * (d + b), 2.0 * m * d * b);
      gemm_nn(Pb, ldb, Ub, d, nullptr, 0, nullptr, Pb + d, ldb, m, d, b, 1.0, 0.0, nullptr, c.st);
    }
    block_orth(c, Pb + d, m, 0, b, ldb, R);
    {
      Prof p(c, P_RESTART, 16.0 * m * b, 0);
      copy_block(Pb + d, ldb, Pb, ldb, m, b, false, c.st);
    }
  }
  if (cycle > maxit) cycle = maxit;
  const bool inplace = outputs_in_place(c, r);
  c.S = dbuf(c, "res_S", (size_t)r);
  c.r = r;
  {
    Prof p(c, P_RESTART, 8.0 * (m + n) * (d + r), 2.0 * (m + n) * d * r);
    // S8 (Eq. 12): V = P_k Vbar[:, :r]; signs (R28) from V, folded into
    // Ubar's columns before S9: U = Pbar_k Ubar[:, :r]
    c.V = out_product(c, "res_V", P, ldp, n, d, Vb, d, r, inplace, &c.ldV);
    double* sgn = signs_of(c, c.V, n, c.ldV, r);
    flip_columns(c.V, n, c.ldV, r, sgn, c.st);
    flip_columns(Ub, d, d, r, sgn, c.st);
    c.U = out_product(c, "res_U", Pb, ldb, m, d, Ub, d, r, inplace, &c.ldU);
    TSVD_CUDA(cudaMemcpyAsync(c.S, Sg, r * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  }
  const double ms = timer.stop();
  prof_harvest(c);
  c.rho = hrho;
  c.have = true;
  c.info = tsvd_info{};
  c.info.cycles = cycle;
  c.info.nconv = nconv;
  c.info.r = r;
  c.info.d = d;
  c.info.b = b;
  c.info.breakdowns = c.breakdowns;
  c.info.replaced = c.replaced;
  c.info.rho_max = rho_max;
  c.info.sigma1 = hs[0];
  c.info.ms_total = ms;
  c.info.launches = g_launches.load() - launches0;
  c.info.svd_sweeps = svdw.max_sweeps;
  c.info.svd_unconverged = svdw.unconverged;
  if (!conv) return TSVD_WARN_NOTCONV;
  return svdw.unconverged ? TSVD_WARN_SVD : TSVD_OK;
}

// SURVEY 8(f) N4 (Eq. 3): the rank is not known in advance but set
// by a threshold on ||A - U_r S_r V_r^T||_2 = sigma_{r+1}.  Reading R33:
// request r + 1 triplets (r = b first), take the smallest r with
// sigma_{r+1} <= tau * sigma_1 whose triplets 1..r+1 all converged
// (rho <= tol); otherwise double r (at most r_max) and solve again from a
// fresh start.  The Krylov dimension is the user's (tsvd_set_krylov_dim) or
// the default for the current request.  Driver-level only: every solve is
// lanczos_solve on the same kernels.
tsvd_status lanczos_threshold(Ctx& c, double tau, int b, double tol, int maxit, int r_max,
                              int* r_out) {
  if (!(tau > 0.0) || tau >= 1.0 || b < 1 || r_max < 1) return TSVD_EINVAL;
  r_max = (int)std::min<int64_t>(r_max, c.ng - 1);
  if (r_max < 1) return TSVD_ESHAPE;
  int req = std::min(b, r_max);
  std::vector<double> hs;
  for (;;) {
    const int want = req + 1;
    const tsvd_status st = lanczos_solve(c, want, b, tol, maxit);
    if (st < 0) return st;
    hs.resize(want);
    TSVD_CUDA(cudaMemcpyAsync(hs.data(), c.S, want * sizeof(double), cudaMemcpyDeviceToHost,
                              c.st));
    TSVD_CUDA(cudaStreamSynchronize(c.st));
    int found = -1;
    for (int r = 1; r < want && c.rho[r - 1] <= tol; ++r) {
      if (c.rho[r] > tol) break;                      // sigma_{r+1} itself not converged
      if (hs[r] <= tau * hs[0]) {
        found = r;
        break;
      }
    }
    if (found > 0 || req >= r_max) {
      const int r = found > 0 ? found : req;
      c.r = r;                                          // tsvd_get: first r columns
      c.info.r = r;
      c.rho.resize(r);
      if (r_out) *r_out = r;
      return found > 0 ? TSVD_OK : TSVD_WARN_NOTCONV;
    }
    req = std::min(2 * req, r_max);
  }
}

tsvd_status rsvd_solve(Ctx& c, int r, int p, int q) {
  const int64_t m = c.m, n = c.n;  // this rank's rows (single GPU: all)
  DeferredGuard guard(c);
  if (r < 1 || p < 0 || q < 0) return TSVD_EINVAL;
  const int l = r + p;
  if (l > c.ng || l > kSmallSvdMaxD) return TSVD_ESHAPE;
  if (!c.start.empty() && (c.start_rows != n || c.start_cols != l)) return TSVD_ESHAPE;
  const int bq = std::min(std::max(1, c.b_qr), 32);
  c.have = false;
  c.breakdowns = 0;
  c.replaced = 0;
  c.draw_next = 1;
  const int64_t launches0 = g_launches.load();
  EventTimer timer(c.st);

  double* Qb = dbuf(c, "Qbar", (size_t)m * l);
  double* Q = dbuf(c, "Q", (size_t)n * l);
  double* R = dbuf(c, "Rp", (size_t)l * l);
  double* Rb = dbuf(c, "Rbarp", (size_t)l * l);
  double* Ub = dbuf(c, "Ub", (size_t)l * l);
  double* Vb = dbuf(c, "Vb", (size_t)l * l);
  double* Sg = dbuf(c, "Sg", (size_t)l);
  double* jw = dbuf(c, "jacobi_work", small_svd_work(l));
  (void)dbuf(c, "scratch", (size_t)std::max(m, n) * 32);
  (void)dbuf(c, "gram", (size_t)nn_ctas(std::max(m, n), 1) * 32 * 32);

  if (!c.start.empty())
    upload_start(c, Q, n, l, l);
  else
    launch_philox_normal(Q, n, l, l, c.seed, 0, c.n0, c.ng, c.st);   // Q_0 (not orthonormal)
  for (int j = 0; j <= q; ++j) {
    apply(c, false, Q, l, Qb, l, l);                                   // S1
    c.cur_row0 = c.m0;
    c.cur_qtot = c.mg;
    cgs_qr(c, Qb, m, l, l, bq, Rb);                                    // S2
    apply(c, true, Qb, l, Q, l, l);                                    // S3
    c.cur_row0 = c.n0;
    c.cur_qtot = c.ng;
    cgs_qr(c, Q, n, l, l, bq, R);                                      // S4
  }
  {
    Prof p(c, P_SVD, 16.0 * l * l, 0);
    small_svd(R, l, Ub, Sg, Vb, jw, c.st);                             // S5
  }
  const bool inplace = outputs_in_place(c, r);
  c.S = dbuf(c, "res_S", (size_t)r);
  c.r = r;
  {
    Prof p(c, P_RESTART, 8.0 * (m + n) * (l + r), 2.0 * (m + n) * l * r);
    c.V = out_product(c, "res_V", Q, l, n, l, Ub, l, r, inplace, &c.ldV);    // S7
    double* sgn = signs_of(c, c.V, n, c.ldV, r);
    flip_columns(c.V, n, c.ldV, r, sgn, c.st);
    flip_columns(Vb, l, l, r, sgn, c.st);
    c.U = out_product(c, "res_U", Qb, l, m, l, Vb, l, r, inplace, &c.ldU);   // S6
    TSVD_CUDA(cudaMemcpyAsync(c.S, Sg, r * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  }
  double s1 = 0.0;
  unsigned* hsw = reinterpret_cast<unsigned*>(c.hflags + 4);
  TSVD_CUDA(cudaMemcpyAsync(&s1, Sg, sizeof(double), cudaMemcpyDeviceToHost, c.st));
  TSVD_CUDA(cudaMemcpyAsync(hsw, small_svd_sweeps_dev(jw, l), sizeof(unsigned),
                            cudaMemcpyDeviceToHost, c.st));
  const double ms = timer.stop();
  SvdWatch svdw;
  svdw.add(*hsw);
  prof_harvest(c);
  c.rho.clear();
  c.have = true;
  c.info = tsvd_info{};
  c.info.cycles = q + 1;
  c.info.r = r;
  c.info.d = l;
  c.info.b = bq;
  c.info.breakdowns = c.breakdowns;
  c.info.replaced = c.replaced;
  c.info.sigma1 = s1;
  c.info.ms_total = ms;
  c.info.launches = g_launches.load() - launches0;
  c.info.svd_sweeps = svdw.max_sweeps;
  c.info.svd_unconverged = svdw.unconverged;
  return svdw.unconverged ? TSVD_WARN_SVD : TSVD_OK;
}

}  // namespace tsvd
