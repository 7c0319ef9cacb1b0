// Handle state of libtsvd (behind the opaque tsvd_t of include/tsvd.h).
#pragma once

#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "internal.h"

namespace tsvd {
struct LoopGroup;
constexpr int kLoopMaxWorld = 8;
// P_ROWT: the s = 0 passes (Gram of Y, TRSM-as-multiply S T) - rowT_kernel
enum ProfCat { P_APPLY_A = 0, P_APPLY_AT, P_TN, P_NN, P_SMALL, P_SVD, P_RESTART, P_OTHER, P_ROWT,
               P_BESIDE_SVD };
struct ProfRec {
  int cat;
  cudaEvent_t a, b;
  int64_t launches;
  double bytes, flops;
  bool graph_owned = false;  // recorded by a captured graph: not returned to the pool
};

// One Lanczos cycle's block steps captured as a CUDA graph (solvers.cu):
// reused while the key (sizes, buffers, options) is unchanged.
struct CycleGraph {
  int64_t m = -1, n = -1;
  int d = 0, b = 0, s0 = 0, kc = 0, ortho = -1;
  unsigned prof = 0;   // profiling phase mask the graph was captured with
  const void* ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
  uint64_t bufgen = 0;
  int seen = 0;                   // eager runs with this key (capture on the second)
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;           // kernels per replay
  std::vector<ProfRec> prof_recs; // phase events inside the graph
};
}  // namespace tsvd

struct tsvd_ctx {
  // Local sizes: m = rows of A (and of U, Pbar) on this rank, n = this rank's
  // n-shard (rows of V, P).  Single GPU: the whole problem.
  int64_t m = 0, n = 0;
  // multi-GPU; world == 1: mg = m, ng = n, offsets 0, nsh = n
  int world = 1, rank = 0;
  void* comm = nullptr;        // ncclComm_t (or the loopback group)
  tsvd::LoopGroup* loop = nullptr;  // test-only in-process communicator (comm.cu)
  int64_t mg = 0, ng = 0;      // global sizes
  int64_t m0 = 0, n0 = 0;      // global offsets of the local rows / n-shard
  int64_t nsh = 0;             // uniform n-shard size (ceil(ng / world))
  int64_t cur_row0 = 0, cur_qtot = 0;  // rows of the block being orthogonalised (Philox)
  bool dense = false;
  tsvd::Csr A, AT;           // CSR(A), CSR(A^T)
  // multi-GPU (world > 1): CSR(A_g^T) cut at the n-shard boundaries, so
  // A_g^T X is produced one shard at a time and each shard's reduction to its
  // owner (ncclReduce) overlaps the next shard's SpMM (comm_st, events)
  std::vector<tsvd::Csr> ATp;
  cudaStream_t comm_st = nullptr;
  // tsvd_get: V's device->host copy runs on copy_st beside U's (two copy
  // engines on the PCIe link instead of one)
  cudaStream_t copy_st = nullptr;
  cudaEvent_t copy_ev = nullptr;
  // the Jacobi SVD of B_k beside the last m-side orthogonalisation (solvers.cu)
  cudaStream_t svd_st = nullptr;
  cudaEvent_t svd_fork = nullptr, svd_join = nullptr;
  std::vector<cudaEvent_t> comm_ev;
  double* Ad = nullptr;      // dense A, row-major m x n
  int64_t lda = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  uint64_t seed = 0x2403062180ULL;
  uint64_t draw_next = 1;    // Philox draw id of the next breakdown replacement
  int krylov_d = 0;
  int thick_keep = 0;         // N1 thick restart: Ritz vectors kept (0 = Alg. 2 S7)
  int b_qr = 16;
  int ortho = TSVD_ORTHO_CGS_CQR2;  // tsvd_set_ortho (SURVEY 8(f) N2 ablation)
  std::vector<double> start;  // optional exact start block (row-major, dense)
  int64_t start_rows = 0, start_cols = 0;
  // device workspace: named buffers grown on demand, kept across solves
  std::map<std::string, std::pair<void*, size_t>> bufs;
  int* dflags = nullptr;      // device flags
  // Deferred breakdown checks (Lanczos): each orthogonalisation writes its two
  // Cholesky breakdown flags to flag_log[2*flag_slot + {0,1}] and the host
  // reads the whole log once per cycle instead of syncing per call; on a
  // breakdown the cycle is replayed from that call with immediate checks.
  bool deferred = false;
  int* flag_log = nullptr;
  int flag_slot = 0;
  int* hflags = nullptr;      // pinned host mirror (8 ints: [0,4) flags, [4] SVD sweeps)
  // results of the last solve
  double *U = nullptr, *S = nullptr, *V = nullptr;
  int64_t ldU = 0, ldV = 0;   // row pitch of U / V (r, or the basis ld in place)
  int out_mode = 0;           // TSVD_OUT_* (tsvd_set_output_mode)
  int r = 0;
  bool have = false;
  std::vector<double> rho;    // rho_i / sigma_1, i < r (LancSVD)
  tsvd_info info{};
  int breakdowns = 0;         // orthogonalisations that fell back to CGS2
  int replaced = 0;           // dependent columns replaced by Philox draws
  // instrumentation (tsvd_set_profiling)
  bool prof_on = false;
  unsigned prof_mask = 0;                 // phases recorded (bit = phase index)
  int prof_override = -1;                 // >= 0: every phase call counts as this one
  std::vector<tsvd::ProfRec> prof_open;   // recorded, not yet harvested
  std::vector<cudaEvent_t> ev_pool;
  tsvd_prof_entry prof[TSVD_NPROF]{};
  // CUDA graph of a Lanczos cycle (single-GPU handles; tsvd_set_graphs)
  // off by default: measured on C2 (profiles/r02), graph replay of the cycle
  // does not shorten the TTS (the inter-kernel gaps are device-side ramp /
  // tail, not host launch latency); TSVD_GRAPHS=1 or tsvd_set_graphs enables it
  bool graphs = getenv("TSVD_GRAPHS") != nullptr && getenv("TSVD_GRAPHS")[0] == '1';
  bool capturing = false;
  uint64_t bufgen = 0;            // bumped by every (re)allocation of a named buffer
  tsvd::CycleGraph cyc_graph;
};

namespace tsvd {
using Ctx = tsvd_ctx;
// named device buffer of at least `bytes`, contents undefined
void* buf(Ctx& c, const std::string& name, size_t bytes);
inline double* dbuf(Ctx& c, const std::string& name, size_t n) {
  return (double*)buf(c, name, n * sizeof(double));
}
void free_bufs(Ctx& c);

// RAII phase scope: events around everything enqueued while alive.
struct Prof {
  Ctx& c;
  int cat;
  double bytes, flops;
  cudaEvent_t a = nullptr;
  int64_t l0 = 0;
  Prof(Ctx& c_, int cat_, double bytes_, double flops_);
  ~Prof();
};
void prof_harvest(Ctx& c);   // after a stream sync: fold records into c.prof
void cycle_graph_reset(Ctx& c);  // drop the captured Lanczos-cycle graph
void prof_release(Ctx& c);

// building blocks (blocks.cu).  All blocks are row-major with leading
// dimension ld; "basis" holds P in columns [0, s) and the block Y being
// orthogonalised in columns [s, s+w).
int cholqr2(Ctx& c, double* Y, int64_t q, int w, int64_t ld, double* R);
// need_h = false: the caller discards H (LancSVD, reading R17), so S12's
// H += Hbar L^T is skipped (H still holds the first projection P^T Y).
int cgs_cqr2(Ctx& c, double* basis, int64_t q, int s, int w, int64_t ld, double* H,
             double* R, bool need_h = true);
void cgs2(Ctx& c, double* basis, int64_t q, int s, int w, int64_t ld, double* H, double* R);
int cgs_qr(Ctx& c, double* Y, int64_t q, int l, int64_t ld, int bq, double* R);
// any-width LancSVD block orthogonalisation (32-column panels above 32)
int block_orth(Ctx& c, double* basis, int64_t q, int s, int b, int64_t ld, double* R);
void apply(Ctx& c, bool trans, const double* X, int64_t ldx, double* Y, int64_t ldy, int w);

// collectives (comm.cu); no-ops / errors when world == 1 / NCCL missing
bool nccl_available();
void nccl_unique_id(void* out128);
void comm_init(Ctx& c, const void* id128, int rank, int world);
void comm_destroy(Ctx& c);
void allreduce_sum(Ctx& c, double* buf, size_t count);
void reduce_scatter_sum(Ctx& c, const double* send, double* recv, size_t recv_count);
void all_gather(Ctx& c, const double* send, double* recv, size_t send_count);
// sum of every rank's send (count) into recv on rank `root`, ordered on `st`
void reduce_sum_to(Ctx& c, const double* send, double* recv, size_t count, int root,
                   cudaStream_t st);
LoopGroup* loop_group_create(int world);
void loop_group_destroy(LoopGroup* g);
void loop_join(Ctx& c, LoopGroup* g, int rank);

// explicit residuals of the last solve (residual.cu):
// e[i] = ||A v_i - s_i u_i|| / s_1, rel[i] = ... / s_i (host arrays, may be NULL)
void residuals(Ctx& c, double* e_host, double* rel_host);

// solvers (solvers.cu)
tsvd_status lanczos_solve(Ctx& c, int r, int b, double tol, int maxit);
tsvd_status rsvd_solve(Ctx& c, int r, int p, int q);
tsvd_status lanczos_threshold(Ctx& c, double tau, int b, double tol, int maxit, int r_max,
                              int* r_out);
}  // namespace tsvd
