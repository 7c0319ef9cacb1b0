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

#include <algorithm>
#include <condition_variable>
#include <mutex>
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
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int,
                         ncclComm_t, cudaStream_t) = nullptr;
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
  a.Reduce = (decltype(a.Reduce))dlsym(h, "ncclReduce");
  a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.ReduceScatter &&
         a.AllGather && a.Reduce;
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
  if (c.loop) {  // the group belongs to the caller (tsvd_loopback_destroy)
    c.loop = nullptr;
    c.comm = nullptr;
    return;
  }
  if (c.comm && api().ok) api().CommDestroy((ncclComm_t)c.comm);
  c.comm = nullptr;
}

// ------------------------------------------------------------- loopback --
// In-process communicator for tests: `world` handles on ONE device, driven
// from `world` host threads, exchange through device memory instead of NCCL.
// It runs the library's complete multi-GPU code path (row shards, n-shard
// padding, Philox row offsets, all-reduced Grams, gathered sign rule) at
// world > 1 on a single GPU.  Every collective is two host barriers and
// cross-stream events: ranks publish their buffers and a "ready" event,
// each rank's stream waits for all ready events, a kernel on its stream
// reads every rank's buffer (plain device pointers: same GPU) and writes its
// own result, and a second barrier + "done" events keep every send buffer
// alive until all ranks have read it.  Sums run over ranks in rank order.
struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  uint64_t gen = 0;
  std::vector<const double*> send;
  std::vector<cudaEvent_t> ready, done;
};

LoopGroup* loop_group_create(int world) {
  if (world < 1 || world > kLoopMaxWorld) throw Error{TSVD_EINVAL, "loopback world out of range"};
  auto* g = new LoopGroup();
  g->world = world;
  g->send.assign(world, nullptr);
  g->ready.assign(world, nullptr);
  g->done.assign(world, nullptr);
  for (int r = 0; r < world; ++r) {
    TSVD_CUDA(cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming));
    TSVD_CUDA(cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
  }
  return g;
}

void loop_group_destroy(LoopGroup* g) {
  if (!g) return;
  for (auto e : g->ready) if (e) cudaEventDestroy(e);
  for (auto e : g->done) if (e) cudaEventDestroy(e);
  delete g;
}

static void loop_barrier(LoopGroup& g) {
  std::unique_lock<std::mutex> lk(g.mu);
  const uint64_t my = g.gen;
  if (++g.count == g.world) {
    g.count = 0;
    ++g.gen;
    g.cv.notify_all();
  } else {
    g.cv.wait(lk, [&] { return g.gen != my; });
  }
}

struct LoopPtrs {
  const double* p[kLoopMaxWorld];
};

// out[i] = sum_k src_k[off + i] (k in rank order)
__global__ void loop_sum_kernel(LoopPtrs src, int world, size_t off, size_t count,
                                double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = src.p[0][off + i];
    for (int k = 1; k < world; ++k) s += src.p[k][off + i];
    out[i] = s;
  }
}

// out[k * count + i] = src_k[i]
__global__ void loop_gather_kernel(LoopPtrs src, int world, size_t count, double* __restrict__ out) {
  const size_t total = (size_t)world * count;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x)
    out[t] = src.p[t / count][t % count];
}

template <class F>
static void loop_collective(Ctx& c, const double* send, F&& body, cudaStream_t st = nullptr) {
  LoopGroup& g = *c.loop;
  const int r = c.rank;
  if (!st) st = c.st;
  g.send[r] = send;
  TSVD_CUDA(cudaEventRecord(g.ready[r], st));
  loop_barrier(g);
  for (int k = 0; k < g.world; ++k)
    if (k != r) TSVD_CUDA(cudaStreamWaitEvent(st, g.ready[k], 0));
  LoopPtrs ptrs{};
  for (int k = 0; k < g.world; ++k) ptrs.p[k] = g.send[k];
  body(ptrs);
  TSVD_CUDA(cudaEventRecord(g.done[r], st));
  loop_barrier(g);  // every rank has read every send buffer (on its stream)
  for (int k = 0; k < g.world; ++k)
    if (k != r) TSVD_CUDA(cudaStreamWaitEvent(st, g.done[k], 0));
}

static unsigned loop_grid(size_t n) {
  return (unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 8));
}

void loop_join(Ctx& c, LoopGroup* g, int rank) {
  c.loop = g;
  c.comm = g;  // non-null: the handle takes the multi-GPU code path
}

// Handles created through tsvd_create_*_dist always run the collectives (also
// with a single rank, which exercises the multi-GPU path on one GPU).
void allreduce_sum(Ctx& c, double* buf, size_t count) {
  if (!c.comm || count == 0) return;
  if (c.loop) {
    // in place: sum into a private buffer, copy back after every rank has read
    double* tmp = dbuf(c, "loop_tmp", count);
    loop_collective(c, buf, [&](const LoopPtrs& p) {
      loop_sum_kernel<<<loop_grid(count), 256, 0, c.st>>>(p, c.loop->world, 0, count, tmp);
      TSVD_CHECK_LAUNCH();
    });
    TSVD_CUDA(cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    return;
  }
  check(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c.comm, c.st),
        "ncclAllReduce");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void reduce_scatter_sum(Ctx& c, const double* send, double* recv, size_t recv_count) {
  if (c.loop) {
    loop_collective(c, send, [&](const LoopPtrs& p) {
      loop_sum_kernel<<<loop_grid(recv_count), 256, 0, c.st>>>(
          p, c.loop->world, (size_t)c.rank * recv_count, recv_count, recv);
      TSVD_CHECK_LAUNCH();
    });
    return;
  }
  check(api().ReduceScatter(send, recv, recv_count, ncclFloat64, ncclSum, (ncclComm_t)c.comm,
                            c.st),
        "ncclReduceScatter");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void reduce_sum_to(Ctx& c, const double* send, double* recv, size_t count, int root,
                   cudaStream_t st) {
  if (c.loop) {
    loop_collective(c, send, [&](const LoopPtrs& p) {
      if (c.rank == root) {
        loop_sum_kernel<<<loop_grid(count), 256, 0, st>>>(p, c.loop->world, 0, count, recv);
        TSVD_CHECK_LAUNCH();
      }
    }, st);
    return;
  }
  check(api().Reduce(send, recv, count, ncclFloat64, ncclSum, root, (ncclComm_t)c.comm, st),
        "ncclReduce");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void all_gather(Ctx& c, const double* send, double* recv, size_t send_count) {
  if (c.loop) {
    loop_collective(c, send, [&](const LoopPtrs& p) {
      loop_gather_kernel<<<loop_grid(send_count * c.loop->world), 256, 0, c.st>>>(
          p, c.loop->world, send_count, recv);
      TSVD_CHECK_LAUNCH();
    });
    return;
  }
  check(api().AllGather(send, recv, send_count, ncclFloat64, (ncclComm_t)c.comm, c.st),
        "ncclAllGather");
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace tsvd
