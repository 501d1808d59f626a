// Multi-GPU target sharding.
//
// The reference MVM (transform.cpp:184-204) splits work over CPU threads by
// node chunks and merges per-thread z. Across GPUs the natural split is by
// TARGET: every rank holds the full plan (tree, sets, tables; cheap), owns a
// contiguous, cost-balanced range [lo, hi) of tree positions, and
//   1. S2M: builds partial node moments from the sources it owns,
//   2. exchange: sum of the moment tables over ranks (nodes x P doubles;
//      3 MB at cfg2) -- the only data-path collective,
//   3. near + M2T: evaluates every interaction whose TARGET it owns (the
//      near-field sources are replicated, so no other exchange),
//   4. scatter: z for its own targets (zeros elsewhere); the host sums z over
//      ranks when every rank needs all of z.
// Because the interaction lists are ascending position lists per node, the
// owned part of every list is one contiguous sub-range (two binary searches),
// so a shard is just a re-tiling of the same kernels.
//
// Cut placement balances an estimated per-target cost: a near pair (t, leaf l)
// costs |l| kernel evaluations; a far pair (t, node) costs farPairWeight(P)
// evaluations (measured on cfg2: one M2T pair ~ 17 near evaluations at P=84).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <numeric>

#include "plan.hpp"

namespace fktb {
namespace {

__global__ void shard_cost_kernel(const long long* off, const uint32_t* pos, const uint32_t* begin, const uint32_t* end,
                                  int nearMode, unsigned long long farWeight, unsigned long long* cost) {
  const int node = blockIdx.x;
  const long long a = off[node], b = off[node + 1];
  if (a == b) return;
  const unsigned long long w = nearMode ? static_cast<unsigned long long>(end[node] - begin[node]) : farWeight;
  for (long long i = a + threadIdx.x; i < b; i += blockDim.x) atomicAdd(cost + pos[i], w);
}

__device__ long long lower_bound_pos(const uint32_t* pos, long long a, long long b, uint32_t v) {
  while (a < b) {
    const long long m = (a + b) >> 1;
    if (pos[m] < v)
      a = m + 1;
    else
      b = m;
  }
  return a;
}

__global__ void subrange_kernel(const long long* off, const uint32_t* pos, int nodes, uint32_t lo, uint32_t hi,
                                long long* out) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nodes) return;
  const long long a = off[node], b = off[node + 1];
  out[2 * node] = lower_bound_pos(pos, a, b, lo);
  out[2 * node + 1] = lower_bound_pos(pos, a, b, hi);
}

void subranges(const DeviceTree& t, bool far, uint32_t lo, uint32_t hi, std::vector<long long>& out) {
  DeviceBuffer<long long> d(static_cast<size_t>(2) * t.nodes);
  subrange_kernel<<<(t.nodes + 127) / 128, 128, 0, t.stream>>>(far ? t.dFarOff.get() : t.dNearOff.get(),
                                                                 far ? t.dFarPos.get() : t.dNearPos.get(), t.nodes, lo,
                                                                 hi, d.get());
  FKTB_CUDA(cudaGetLastError());
  out.resize(static_cast<size_t>(2) * t.nodes);
  FKTB_CUDA(cudaMemcpyAsync(out.data(), d.get(), d.bytes(), cudaMemcpyDeviceToHost, t.stream));
  FKTB_CUDA(cudaStreamSynchronize(t.stream));
}

}  // namespace

unsigned long long farPairWeight(int P) { return static_cast<unsigned long long>(std::max(1, P / 5)); }

std::vector<uint32_t> shardCuts(const DeviceTree& t, int P, int shards) {
  const int n = t.n;
  std::vector<uint32_t> cuts(static_cast<size_t>(shards) + 1, 0);
  cuts[static_cast<size_t>(shards)] = static_cast<uint32_t>(n);
  if (shards == 1) return cuts;
  DeviceBuffer<unsigned long long> dCost(static_cast<size_t>(n));
  FKTB_CUDA(cudaMemsetAsync(dCost.get(), 0, dCost.bytes(), t.stream));
  shard_cost_kernel<<<t.nodes, 256, 0, t.stream>>>(t.dNearOff.get(), t.dNearPos.get(), t.dBegin.get(), t.dEnd.get(), 1,
                                                   0, dCost.get());
  FKTB_CUDA(cudaGetLastError());
  shard_cost_kernel<<<t.nodes, 256, 0, t.stream>>>(t.dFarOff.get(), t.dFarPos.get(), t.dBegin.get(), t.dEnd.get(), 0,
                                                   farPairWeight(P), dCost.get());
  FKTB_CUDA(cudaGetLastError());
  // cumulative cost over tree positions; cuts at any position (not only leaf
  // boundaries: a leaf split between ranks just has its sources' moments
  // summed by the exchange and its near list sub-ranged by target)
  DeviceBuffer<unsigned long long> dCum(static_cast<size_t>(n));
  {
    size_t bytes = 0;
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, dCost.get(), dCum.get(), n, t.stream));
    DeviceBuffer<unsigned char> temp(bytes + 1);
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, dCost.get(), dCum.get(), n, t.stream));
    FKTB_CUDA(cudaStreamSynchronize(t.stream));
  }
  std::vector<unsigned long long> cum(static_cast<size_t>(n));
  FKTB_CUDA(cudaMemcpyAsync(cum.data(), dCum.get(), dCum.bytes(), cudaMemcpyDeviceToHost, t.stream));
  FKTB_CUDA(cudaStreamSynchronize(t.stream));
  const unsigned long long total = cum.back();
  for (int s = 1; s < shards; ++s) {
    // the boundary after position p carries cum[p]: the one closest to s/shards of the total
    const double goal = static_cast<double>(total) * s / shards;
    size_t p = static_cast<size_t>(std::lower_bound(cum.begin(), cum.end(), static_cast<unsigned long long>(goal)) -
                                   cum.begin());
    if (p >= static_cast<size_t>(n)) p = static_cast<size_t>(n) - 1;
    uint32_t c = static_cast<uint32_t>(p + 1);
    if (p > 0 && goal - static_cast<double>(cum[p - 1]) < static_cast<double>(cum[p]) - goal) c = static_cast<uint32_t>(p);
    cuts[static_cast<size_t>(s)] = std::max(c, cuts[static_cast<size_t>(s) - 1]);
  }
  return cuts;
}

std::vector<uint32_t> shardCutsFromLeaves(const std::vector<std::pair<uint32_t, unsigned long long>>& leafEnd, int shards,
                                          uint32_t n) {
  std::vector<uint32_t> cuts(static_cast<size_t>(shards) + 1, 0);
  cuts[static_cast<size_t>(shards)] = n;
  const unsigned long long total = leafEnd.empty() ? 0 : leafEnd.back().second;
  size_t li = 0;
  for (int s = 1; s < shards; ++s) {
    // first leaf boundary whose cumulative cost reaches s/shards of the total
    const double goal = static_cast<double>(total) * s / shards;
    while (li < leafEnd.size() && static_cast<double>(leafEnd[li].second) < goal) ++li;
    uint32_t c = li < leafEnd.size() ? leafEnd[li].first : n;
    // the boundary just before may be closer to the goal
    if (li > 0 && li < leafEnd.size()) {
      const double over = static_cast<double>(leafEnd[li].second) - goal;
      const double under = goal - static_cast<double>(leafEnd[li - 1].second);
      if (under < over) c = leafEnd[li - 1].first;
    }
    cuts[static_cast<size_t>(s)] = std::max(c, cuts[static_cast<size_t>(s) - 1]);
  }
  return cuts;
}

void setShard(DevicePlan& plan, int shard, int shards) {
  if (shards < 1 || shard < 0 || shard >= shards) throw std::invalid_argument("shard must satisfy 0 <= shard < shards");
  const DeviceTree& t = *plan.tree;
  const std::vector<uint32_t> cuts = shardCuts(t, plan.P, shards);
  plan.shard = shard;
  plan.shards = shards;
  plan.shardLo = cuts[static_cast<size_t>(shard)];
  plan.shardHi = cuts[static_cast<size_t>(shard) + 1];
  plan.cuts = cuts;
  if (shards == 1) {
    plan.farSub.clear();
    plan.nearSub.clear();
  } else {
    subranges(t, true, plan.shardLo, plan.shardHi, plan.farSub);
    subranges(t, false, plan.shardLo, plan.shardHi, plan.nearSub);
  }
  rebuildTiles(plan);
}

}  // namespace fktb
