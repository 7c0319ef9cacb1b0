// NCCL plumbing for the row-partitioned multi-GPU path.
//
// NCCL is resolved at run time with dlopen/dlsym so libtsvd.so has no link
// dependency on a particular NCCL build: inside a PyTorch process the
// already-loaded libnccl.so.2 (torch's) is reused (RTLD_NOLOAD first), else
// the system one is opened.  Only the types come from <nccl.h>.
//
// Collectives used per Lanczos block step (all on the handle's stream):
//   reduce-scatter  A_g^T Qbar_i partials (n x b)   -> this rank's n-shard
//   all-reduce      H, Hbar (s x b), W, Wbar (b x b) (sum of row-shard partials)
//   all-gather      Q_i (n-shards -> full n x b) before A_g Q_i
// B_k, the Jacobi SVD, rho and the restart decision are replicated on every
// rank from bitwise-identical all-reduced inputs.
#include <dlfcn.h>
#include <nccl.h>

#include "ctx.h"

namespace tsvd {

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
  a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
  a.ReduceScatter = (decltype(a.ReduceScatter))dlsym(h, "ncclReduceScatter");
  a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
  a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.ReduceScatter &&
         a.AllGather;
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw Error{TSVD_ENCCL, std::string(what) + ": " + s};
  }
}
}  // namespace

bool nccl_available() { return api().ok; }

void nccl_unique_id(void* out128) {
  if (!api().ok) throw Error{TSVD_ENCCL, "libnccl.so.2 not found"};
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
}

void comm_init(Ctx& c, const void* id128, int rank, int world) {
  if (!api().ok) throw Error{TSVD_ENCCL, "libnccl.so.2 not found"};
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t comm;
  check(api().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
  c.comm = comm;
}

void comm_destroy(Ctx& c) {
  if (c.comm && api().ok) api().CommDestroy((ncclComm_t)c.comm);
  c.comm = nullptr;
}

// Handles created through tsvd_create_*_dist always run the collectives (also
// with a single rank, which exercises the multi-GPU path on one GPU).
void allreduce_sum(Ctx& c, double* buf, size_t count) {
  if (!c.comm || count == 0) return;
  check(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c.comm, c.st),
        "ncclAllReduce");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void reduce_scatter_sum(Ctx& c, const double* send, double* recv, size_t recv_count) {
  check(api().ReduceScatter(send, recv, recv_count, ncclFloat64, ncclSum, (ncclComm_t)c.comm,
                            c.st),
        "ncclReduceScatter");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void all_gather(Ctx& c, const double* send, double* recv, size_t send_count) {
  check(api().AllGather(send, recv, send_count, ncclFloat64, (ncclComm_t)c.comm, c.st),
        "ncclAllGather");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace tsvd
