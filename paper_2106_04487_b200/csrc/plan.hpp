// Host-side plan structures (product code). A DeviceTree owns the GPU copy of
// the partition tree and its interaction sets; a DevicePlan adds the
// expansion tables and the MVM workspaces. See DESIGN.md §2 for the HBM
// layout.
#ifndef FKTB_PLAN_HPP
#define FKTB_PLAN_HPP

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "fkt_device_types.h"
#include "tables.hpp"

namespace fktb {

template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) { resize(n); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_), cap_(o.cap_) {
    o.p_ = nullptr;
    o.n_ = o.cap_ = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      cap_ = o.cap_;
      o.p_ = nullptr;
      o.n_ = o.cap_ = 0;
    }
    return *this;
  }
  // Keeps the allocation when it is large enough (re-plans reuse buffers:
  // cudaMalloc / cudaFree of hundreds of MB synchronise the device and cost
  // milliseconds); the contents are NOT preserved either way.
  // A buffer that has to GROW gets 1/8 headroom (list sizes drift between
  // rebuilds on moving points; the first allocation is exact).
  void resize(std::size_t n) {
    if (n <= cap_) {
      n_ = n;
      return;
    }
    const std::size_t c = cap_ ? n + n / 8 : n;
    release();
    if (c) FKTB_CUDA(cudaMalloc(&p_, c * sizeof(T)));
    n_ = n;
    cap_ = c;
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = cap_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  std::size_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0, cap_ = 0;
};

// Partition tree + interaction sets resident in HBM.
struct DeviceTree {
  int n = 0, d = 0, leafCapacity = 0;
  double theta = 0.0;
  bool hasSets = false;
  int depth = 0;

  // Device: permuted coordinates SoA (pc[a*n + pos]), permutation pos->orig.
  DeviceBuffer<double> pc;
  DeviceBuffer<uint32_t> order;

  // Host node arrays in reference pre-order numbering (tree.cpp:41-171).
  int nodes = 0;
  std::vector<uint32_t> begin, end;
  std::vector<int> left, right;
  std::vector<double> boxLo, boxHi, center, radius;  // d per node for box/center

  // Device node arrays (pre-order).
  DeviceBuffer<double> dCenter, dLimit2;
  DeviceBuffer<int> dLeft, dRight;
  DeviceBuffer<uint32_t> dBegin, dEnd;

  // Interaction sets as node-major CSR over PERMUTED positions, ascending
  // (tree.cpp:173-213 restated point-wise on the GPU).
  long long farTotal = 0, nearTotal = 0;
  std::vector<long long> farOff, nearOff;  // host copies, nodes + 1
  DeviceBuffer<long long> dFarOff, dNearOff;
  DeviceBuffer<uint32_t> dFarPos, dNearPos;

  // Build temporaries kept across rebuilds (fkt_plan_rebuild: same n, d).
  struct Scratch {
    DeviceBuffer<double> x, tc, lo, hi, c, r;
    DeviceBuffer<uint32_t> torder, farNode, farPos, nearNode, nearPos, keysOut;
    DeviceBuffer<int> segB, segE, mid, narOut, itemLower, itemLowPre, itemUpPre, wideB, wideE, wideOut, segItem;
    DeviceBuffer<int> farCnt, nearCnt;
    DeviceBuffer<long long> farStart, nearStart;
    DeviceBuffer<unsigned char> temp;
    DeviceBuffer<int4> items;
    DeviceBuffer<unsigned char> wide;  // WideSeg records
  } scratch;

  cudaStream_t stream = nullptr;
};

// Build the tree for `x` (row-major n x d, host) on `stream`.
// devX: the same coordinates already on the device (row-major), else hostX is copied
void buildTreeGpu(DeviceTree& t, const double* hostX, int n, int d, int leafCapacity, cudaStream_t stream,
                  const double* devX = nullptr);
void computeSetsGpu(DeviceTree& t, double theta);

// Host materialisation of the sets in the reference's form: original point
// indices, ascending per node.
void materializeSets(const DeviceTree& t, bool far, std::vector<long long>& off, std::vector<uint32_t>& idx);

// ---------------------------------------------------------------------------
struct PlanOptions {
  int p = 4;
  double theta = 0.75;
  int leafCapacity = 512;
  int compression = 0;  // 0 auto, 1 on, 2 off
  bool eagerOperators = true;
  bool barnesHut = false;
  int threads = 0;
  bool hasDiagonal = false;
  double diagonal = 0.0;
  int nearPrecision = 64;  // 64: FP64 near field; 32: FP32 fast mode (near32.cu)
  bool deterministic = false;  // bitwise reproducible z (det.cu)
};

struct DetIndex {
  DeviceBuffer<uint32_t> idx;
  DeviceBuffer<long long> groupOff;
};

struct DevicePlan {
  int n = 0, d = 0;
  PlanOptions options;
  KernelSpec kernel;
  std::unique_ptr<DeviceTree> tree;
  bool compressed = false;
  std::vector<RadialFactor> factors;
  std::unique_ptr<HarmonicStructure> harmonics;
  int P = 0, H = 0;

  std::unique_ptr<FktbFarParams> far;   // kernel-parameter tables
  DeviceBuffer<double> dHScale;          // per harmonic: Z_k * norm_h^2
  DeviceBuffer<int> dChainG, dChainC, dChainPh;  // generic runtime chain table
  std::vector<FktbTile> farTilesHost, nearTilesHost, s2mTilesHost;
  DeviceBuffer<FktbTile> dFarTiles, dNearTiles, dS2mTiles;
  DeviceBuffer<double> dMoments;         // nodes x P x nrhsCap
  DeviceBuffer<double> dX;               // original coordinates, row-major (dense paths)
  DeviceBuffer<double> dYp, dZp;         // permuted workspaces (n x nrhsCap)
  DeviceBuffer<double> dYio, dZio;       // staging for host-buffer multiplies
  // host-buffer multiplies (hostio.cu): copy streams, group events, pinned
  // bounce buffers for pageable y / z
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t evIo[4] = {};
  void* bounceIn = nullptr;
  void* bounceOut = nullptr;
  size_t bounceBytes = 0;
  int nrhsCap = 0;
  double planSeconds = 0.0;
  // plan-time phases (seconds): tree, sets, exact tables, tiles, near rows,
  // moment plan, other (fkt_plan_phases)
  double phaseSeconds[7] = {};
  std::mutex mutex;                       // multiply() is serialised per plan
  cudaStream_t stream = nullptr;
  // Far-field side stream: S2M -> M2T run concurrently with the near field.
  cudaStream_t side = nullptr;
  cudaEvent_t evGather = nullptr, evFar = nullptr;
  // Recorded after every multiply / stage on the caller's stream; the next
  // call (on any stream) waits on it, because the workspaces are per plan.
  cudaEvent_t evDone = nullptr;
  bool doneRecorded = false;
  // Monomial-moment S2M (moments.cu) for the compile-time shapes.
  bool useMoments = false;
  int monoCount = 0;
  std::vector<double> hscaleHost, kappaHost;
  DeviceBuffer<double> dMono, dMomT, dMomTT, dShiftCoef;  // dMomTT: T transposed, count x P
  // Cartesian (q-form) M2T of single-RHS multiplies (far.cu m2t_cart): the
  // per-node coefficient count (0: not used by this plan) and the map from the
  // monomial moments, transposed (count x cartP)
  int cartP = 0;
  DeviceBuffer<double> dCartTT;
  DeviceBuffer<double> dM2tScale;  // P: d = 3 fused M2T moment scale 1 / (n! kappa_n) (far.cu m2t_fused)
  int shiftEntries = 0;
  DeviceBuffer<int> dShiftOff, dShiftB, dShiftG, dMonoExps, dLevelNodes, dFarNodes;
  std::vector<FktbTile> p2mTilesHost;
  DeviceBuffer<FktbTile> dP2mTiles;
  std::vector<int> levelOff;     // internal nodes grouped by depth: [levelOff[l], levelOff[l+1])
  // Narrow top of the tree: internal nodes shallower than m2mTop (8) get their
  // moments in ONE launch, straight from their frontier (descendants at depth
  // m2mTop, or leaves above it) by composite shifts; (node, frontier) pairs.
  int m2mTop = 0;
  int topPairs = 0;
  DeviceBuffer<int> dTopPairs;
  std::vector<int> farNodesHost; // nodes with a non-empty far set
  // Streaming near field (near.cu near_stream): geometry rows (n x GS, plan
  // time), the factored Gaussian's per-source weight factor, the per-pass
  // source-major weights, two tile-claim counters; near tiles are ordered
  // Gram form first (nearGramTileCount of them).
  bool nearRowsBuilt = false;
  long long nearGramTileCount = 0;
  DeviceBuffer<double> dNearRows, dNearFac, dNearW;
  DeviceBuffer<int> dNearCounter;
  // Target shard (shard.cu): owned tree positions [shardLo, shardHi) and the
  // owned sub-range [sub[2b], sub[2b+1]) of every node's far / near list
  // (empty = whole lists).
  int shard = 0, shards = 1;
  uint32_t shardLo = 0, shardHi = 0;
  std::vector<uint32_t> cuts;  // every rank's range: [cuts[r], cuts[r + 1])
  std::vector<long long> farSub, nearSub;
  // Barnes-Hut plans (bh.cu): per-node centres of mass, nodes x d.
  DeviceBuffer<double> dCom;
  // Captured CUDA graphs of the whole MVM, per (y, z, nrhs, stream); replayed
  // on repeat calls (launch-bound small problems). Cleared on reallocation.
  // Bounded: callers that pass fresh buffers every call would otherwise grow
  // it without limit; the least recently launched graph is dropped past
  // kMaxGraphs.
  static constexpr int kMaxGraphs = 8;
  std::map<std::tuple<const void*, const void*, int, cudaStream_t>, std::pair<cudaGraphExec_t, unsigned long long>>
      graphs;
  unsigned long long graphClock = 0;
  bool useGraphs = true;
  // sharded multiplies (multigpu.cu): graph per (y, z, nrhs, stream) with its
  // communicator and the communicator epoch it was captured in
  struct ShardedGraph {
    cudaGraphExec_t exec;
    void* comm;
    unsigned long long epoch;
  };
  std::map<std::tuple<const void*, const void*, int, cudaStream_t>, ShardedGraph> shardedGraphs;
  // Deterministic mode (det.cu): per list, the per-target index into the
  // partials (sliced by groups of 32 targets, group offsets); the partials of
  // one pass ([entry][rhs], slotsTotal = near + far entries), z_far, the
  // per-tile S2M partials and their node ranges.
  bool detBuilt = false;
  long long slotsTotal = 0;
  DetIndex detNear, detFar;
  DeviceBuffer<double> dPart, dTilePart, dZf;
  DeviceBuffer<int> dDetTileRanges;
  int detTileNodes = 0;
};

enum { kPhaseTree = 0, kPhaseSets, kPhaseTables, kPhaseTiles, kPhaseNearRows, kPhaseMoments, kPhaseOther, kPhaseCount };

std::unique_ptr<DevicePlan> createPlan(int n, int d, const double* hostX, const KernelSpec& kernel,
                                       const PlanOptions& options);
void destroyPlan(DevicePlan* plan);
// Same plan, new coordinates of the same n points (moving points).
// x: row-major n x d, on the host or (onDevice) in device memory
void rebuildPlan(DevicePlan& plan, const double* x, bool onDevice = false);
// Multi-GPU (multigpu.cu): NCCL communicators (dlopen'd libnccl) and the
// sharded MVM with both exchanges in one graph.
void ncclUniqueIdBytes(char* out128);
void* ncclCommCreate(const char* idBytes, int nranks, int rank);
void ncclCommRelease(void* comm);
void multiplySharded(DevicePlan& plan, const double* y, double* z, int nrhs, void* comm, cudaStream_t stream);
void clearShardedGraphs(DevicePlan& plan);
// Doubles per (rhs, node) row of dMoments in an nrhs-column pass: single-RHS
// passes of plans with a Cartesian M2T store its coefficients instead of the
// (k, s, h) moments.
inline bool cartPass(const DevicePlan& plan, int nrhs) { return plan.cartP > 0 && nrhs == 1; }
inline int momentStride(const DevicePlan& plan, int nrhs) { return cartPass(plan, nrhs) ? plan.cartP : plan.P; }
inline int momentStrideMax(const DevicePlan& plan) { return plan.cartP > plan.P ? plan.cartP : plan.P; }
// z = K y for nrhs column-major right-hand sides; y, z device pointers.
void multiplyDevice(DevicePlan& plan, const double* y, double* z, int nrhs, cudaStream_t stream);
// z = K y on host buffers (pinned or pageable), synchronous (hostio.cu).
void multiplyHost(DevicePlan& plan, const double* y, double* z, int nrhs);
void releaseHostIo(DevicePlan& plan);

// 2^(j/2^bits), j < 2^bits, in device memory (default 64 entries: the far
// kernels; the near field uses kNearExpBits).
const double* expTableDevice(int bits = 6, bool compensated = false);

// Kernel launchers (near.cu, far.cu, dense.cu).
// Multi-GPU target sharding (shard.cu).
void setShard(DevicePlan& plan, int shard, int shards);
std::vector<uint32_t> shardCuts(const DeviceTree& t, int P, int shards);
std::vector<uint32_t> shardCutsFromLeaves(const std::vector<std::pair<uint32_t, unsigned long long>>& leafEnd, int shards,
                                          uint32_t n);
unsigned long long farPairWeight(int P);
void rebuildTiles(DevicePlan& plan);
// Grow the per-nrhs workspaces (moments, permuted y/z) up to one pass;
// clears captured graphs.
void ensureWorkspace(DevicePlan& plan, int nrhs);
// Right-hand sides one pass of the MVM takes (shared-memory bound; multiply
// loops over passes).
constexpr int kMaxRhsPerPass = 64;
int maxRhsPerPass(const DevicePlan& plan);
// Stream ordering between calls on one plan (multiply, stage_device).
void orderAfterPrevious(DevicePlan& plan, cudaStream_t st);
void markDone(DevicePlan& plan, cudaStream_t st);
// Number of this library's kernels one multiply launches (memsets excluded).
long long kernelLaunches(const DevicePlan& plan, int nrhs);

// Barnes-Hut monopole far field (bh.cu).
void buildBarnesHut(DevicePlan& plan);
void launchBHSums(const DevicePlan& plan, const double* yp, double* totals, int nrhs, cudaStream_t stream);
void launchBHFar(const DevicePlan& plan, const double* totals, double* zp, int nrhs, cudaStream_t stream);

// Deterministic mode (det.cu).
void buildDeterministic(DevicePlan& plan);
void buildDetTileRanges(DevicePlan& plan);
ZOut zoutFor(const DevicePlan& plan, double* zp, int nrhs, bool far);
ZOut zoutShift(ZOut o, int r0);
// far = true: z_far from the far partials; false: zp = z_far + the near partials
void launchDetReduce(const DevicePlan& plan, double* zp, int nrhs, bool far, cudaStream_t stream);
void launchDetTileSum(const DevicePlan& plan, const double* part, int PC, int nrhs, double* moments, cudaStream_t stream);
// per-tile S2M partials one launch of nrhs right-hand sides needs (doubles)
size_t detTilePartSize(const DevicePlan& plan, int nrhs);

void launchNear(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t stream);
// Streaming near field: plan-time rows and tile order (near.cu); launches
// per multiply.
void buildNearRows(DevicePlan& plan);
long long nearLaunches(const DevicePlan& plan, int nrhs);
// Near tiles the FP64 near field runs in Gram form (near.cu); the rest run the
// difference form in a second launch.
long long nearGramTiles(const DevicePlan& plan);
bool launchNear32(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t stream);
// FP32 fast mode when requested and available for (kernel, d), else FP64.
void launchNearAny(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t stream);
void launchS2M(const DevicePlan& plan, const double* yp, double* moments, int nrhs, cudaStream_t stream);
bool momentsSupported(int d, int p);
// P2M launches of one multiply with nrhs right-hand sides (moments.cu).
int p2mLaunches(int d, int p, int count, int nrhs);
void launchS2MMoments(const DevicePlan& plan, const double* yp, double* moments, int nrhs, cudaStream_t stream);
// Monomial-moment S2M when the plan has it, else the direct S2M.
void launchS2MAny(const DevicePlan& plan, const double* yp, double* moments, int nrhs, cudaStream_t stream);
void launchM2T(const DevicePlan& plan, const double* moments, double* zp, int nrhs, cudaStream_t stream);
void launchGatherY(const DevicePlan& plan, const double* y, double* yp, int nrhs, cudaStream_t stream);
void launchScatterZ(const DevicePlan& plan, const double* zp, double* z, int nrhs, cudaStream_t stream);
void denseRowsGpu(int n, int d, const double* dX, const FktbKernelDesc& kd, const double* dY, int m,
                  const int64_t* dRows, double* dZ, cudaStream_t stream);

}  // namespace fktb

#endif
