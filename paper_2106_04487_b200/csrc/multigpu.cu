// Multi-GPU MVM in one call: target sharding with the moment
// exchange and the z exchange inside the MVM graph.
//
// The reference parallelises one MVM over CPU threads by node chunks and
// merges their z buffers (transform.cpp:18-35, 184-204). Here every rank (one
// process per GPU) holds the full plan, owns the cost-balanced range
// [lo_r, hi_r) of tree positions (shard.cu) and runs, on its stream:
//
//   main:  gather y -> zero z --------------> near (owned targets) ---+
//   side:            \-> zero moments -> S2M (owned sources)          |
//                         -> all-reduce(moments, sum)  [NCCL]         |
//                         -> M2T (owned targets) -------------------->+
//   main:  broadcast of every rank's owned z range (tree order) [NCCL]
//          -> scatter z (all of z on every rank)
//
// captured once per (y, z, nrhs, stream) as a CUDA graph, so a step is one
// graph launch. NCCL is loaded at run time (dlopen of libnccl.so.2, which
// resolves to the process's copy when torch has loaded one), so the library
// itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "plan.hpp"

namespace fktb {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*commUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.getUniqueId, "ncclGetUniqueId");
    sym(api.commInitRank, "ncclCommInitRank");
    sym(api.commDestroy, "ncclCommDestroy");
    sym(api.commCount, "ncclCommCount");
    sym(api.commUserRank, "ncclCommUserRank");
    sym(api.allReduce, "ncclAllReduce");
    sym(api.broadcast, "ncclBroadcast");
    sym(api.groupStart, "ncclGroupStart");
    sym(api.groupEnd, "ncclGroupEnd");
    sym(api.errorString, "ncclGetErrorString");
  });
  if (!api.error.empty()) throw std::invalid_argument("unsupported on the GPU path (multi-GPU): " + api.error);
  return api;
}

// Bumped by every communicator destroy: a sharded graph captured before it
// may reference a freed communicator whose address a new one reuses, so
// graphs remember the epoch they were captured in and are re-captured.
std::atomic<unsigned long long> g_commEpoch{0};

void ncclCheck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaError(std::string("NCCL error in ") + what + ": " + (nccl().errorString ? nccl().errorString(r) : "?"));
}

// One pass (<= maxRhsPerPass columns) of the sharded MVM.
void enqueueShardedPass(DevicePlan& plan, const double* y, double* z, int nrhs, ncclComm_t comm, cudaStream_t st) {
  const NcclApi& N = nccl();
  const size_t n = static_cast<size_t>(plan.n);
  launchGatherY(plan, y, plan.dYp.get(), nrhs, st);
  FKTB_CUDA(cudaMemsetAsync(plan.dZp.get(), 0, n * nrhs * sizeof(double), st));
  FKTB_CUDA(cudaEventRecord(plan.evGather, st));
  FKTB_CUDA(cudaStreamWaitEvent(plan.side, plan.evGather, 0));
  const size_t mom = static_cast<size_t>(plan.tree->nodes) * momentStride(plan, nrhs) * nrhs;
  FKTB_CUDA(cudaMemsetAsync(plan.dMoments.get(), 0, mom * sizeof(double), plan.side));
  launchS2MAny(plan, plan.dYp.get(), plan.dMoments.get(), nrhs, plan.side);
  ncclCheck(N.allReduce(plan.dMoments.get(), plan.dMoments.get(), mom, ncclFloat64, ncclSum, comm, plan.side),
            "moment all-reduce");
  launchNearAny(plan, plan.dYp.get(), plan.dZp.get(), nrhs, st);
  launchM2T(plan, plan.dMoments.get(), plan.dZp.get(), nrhs, plan.side);
  if (plan.options.deterministic) launchDetReduce(plan, nullptr, nrhs, true, plan.side);
  FKTB_CUDA(cudaEventRecord(plan.evFar, plan.side));
  FKTB_CUDA(cudaStreamWaitEvent(st, plan.evFar, 0));
  if (plan.options.deterministic) launchDetReduce(plan, plan.dZp.get(), nrhs, false, st);
  // every rank's owned z range to every rank (in place: non-owned entries
  // are zero until their owner's broadcast lands)
  ncclCheck(N.groupStart(), "group start");
  for (int r = 0; r < plan.shards; ++r) {
    const size_t lo = plan.cuts[static_cast<size_t>(r)], hi = plan.cuts[static_cast<size_t>(r) + 1];
    if (hi <= lo) continue;
    for (int c = 0; c < nrhs; ++c) {
      double* p = plan.dZp.get() + static_cast<size_t>(c) * n + lo;
      ncclCheck(N.broadcast(p, p, hi - lo, ncclFloat64, r, comm, st), "z broadcast");
    }
  }
  ncclCheck(N.groupEnd(), "group end");
  launchScatterZ(plan, plan.dZp.get(), z, nrhs, st);
}

}  // namespace

void ncclUniqueIdBytes(char* out) {
  ncclUniqueId id;
  ncclCheck(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

void* ncclCommCreate(const char* idBytes, int nranks, int rank) {
  ncclUniqueId id;
  std::memcpy(id.internal, idBytes, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  ncclCheck(nccl().commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  return comm;
}

void ncclCommRelease(void* comm) {
  if (!comm) return;
  nccl().commDestroy(static_cast<ncclComm_t>(comm));
  g_commEpoch.fetch_add(1);
}

void multiplySharded(DevicePlan& plan, const double* y, double* z, int nrhs, void* commPtr, cudaStream_t st) {
  auto comm = static_cast<ncclComm_t>(commPtr);
  int world = 0, rank = 0;
  ncclCheck(nccl().commCount(comm, &world), "ncclCommCount");
  ncclCheck(nccl().commUserRank(comm, &rank), "ncclCommUserRank");
  if (plan.shards != world || plan.shard != rank)
    throw std::invalid_argument("sharded multiply: set the plan's shard to (comm rank, comm size) first");
  ensureWorkspace(plan, nrhs);
  orderAfterPrevious(plan, st);
  const int chunk = maxRhsPerPass(plan);
  const size_t n = static_cast<size_t>(plan.n);
  auto enqueue = [&] {
    for (int r0 = 0; r0 < nrhs; r0 += chunk)
      enqueueShardedPass(plan, y + r0 * n, z + r0 * n, std::min(chunk, nrhs - r0), comm, st);
  };
  if (!plan.useGraphs || st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) {
    enqueue();
    markDone(plan, st);
    return;
  }
  // one graph per (y, z, nrhs, stream, communicator): a step is one launch
  const auto key = std::make_tuple(static_cast<const void*>(y), static_cast<const void*>(z), nrhs, st);
  auto it = plan.shardedGraphs.find(key);
  const unsigned long long epoch = g_commEpoch.load();
  if (it == plan.shardedGraphs.end() || it->second.comm != commPtr || it->second.epoch != epoch) {
    if (it != plan.shardedGraphs.end()) {
      cudaGraphExecDestroy(it->second.exec);
      plan.shardedGraphs.erase(it);
    }
    cudaGraph_t graph = nullptr;
    FKTB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    FKTB_CUDA(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    FKTB_CUDA(e);
    it = plan.shardedGraphs.emplace(key, DevicePlan::ShardedGraph{exec, commPtr, epoch}).first;
  }
  FKTB_CUDA(cudaGraphLaunch(it->second.exec, st));
  markDone(plan, st);
}

void clearShardedGraphs(DevicePlan& plan) {
  for (auto& kv : plan.shardedGraphs) cudaGraphExecDestroy(kv.second.exec);
  plan.shardedGraphs.clear();
}

}  // namespace fktb
