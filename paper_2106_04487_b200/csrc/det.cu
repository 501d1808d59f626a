// Deterministic MVM mode (FktOptions::deterministic; additive, no reference
// option). The reference is bit-reproducible at a fixed thread count because
// it merges its per-thread z buffers in a fixed order (transform.cpp:194-203).
// The default GPU path accumulates z and the moments with FP64 atomics from
// many CTAs and two streams, so the last bits of z vary run to run. Here:
//
//  * every near / far kernel STORES its (target, list entry) result at that
//    entry of a partial array (near entries, then far entries; right-hand
//    sides minor) instead of an atomic: coalesced stores, since a tile's
//    entries are consecutive (common.cuh ZOut);
//  * one thread per target then adds its partials in a fixed order through
//    a per-list index built at plan time, sliced by groups of 32 consecutive
//    targets: slot j of a group is the group's j-th node (ascending) among
//    the nodes whose list holds any of its targets, and lane l of slot j (at
//    off[g] + 32 j + l) the entry of target 32 g + l in that node's list, or
//    a pad. The group's targets in one node's list are consecutive entries,
//    so both the index and the partial reads are coalesced. The far sum runs
//    on the far-field stream right after the M2T (hidden behind the near
//    field), the near sum after the join:
//        z_far[t] = sum over t's far entries, ascending node
//        z[t]     = z_far[t] + sum over t's near entries, ascending leaf;
//  * node moments: one P2M tile per leaf, per-level M2M only (plan.cu), and
//    per-tile direct-S2M partials summed in tile order (tile_sum_kernel).
//
// HBM (cfg2): partials 8 B per entry and right-hand side (1.0 GB), the
// sliced index ~4.5 B per entry (0.57 GB).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <limits>
#include <vector>

#include "plan.hpp"

namespace fktb {
namespace {

__global__ void fill_kernel(uint32_t* v, long long n, uint32_t x) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = x;
}

__global__ void iota_kernel(uint32_t* v, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<uint32_t>(i);
}

// key of every list entry: (target group, node)
__global__ void entry_key_kernel(const long long* off, const uint32_t* pos, unsigned long long* key) {
  const int b = blockIdx.x;
  for (long long e = off[b] + threadIdx.x; e < off[b + 1]; e += blockDim.x)
    key[e] = (static_cast<unsigned long long>(pos[e] >> 5) << 32) | static_cast<unsigned>(b);
}

__global__ void new_slot_kernel(const unsigned long long* key, long long m, long long* flag) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) flag[i] = i == 0 || key[i] != key[i - 1];
}

// C = inclusive count of distinct (group, node) keys: the group's first
// slot number, and (second pass) its slot count x 32
__global__ void group_first_kernel(const unsigned long long* key, const long long* C, long long m, long long* first) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long g = key[i] >> 32;
  if (i == 0 || (key[i - 1] >> 32) != g) first[g] = C[i];
}

__global__ void group_width_kernel(const unsigned long long* key, const long long* C, long long m, const long long* first,
                                   long long* width) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long g = key[i] >> 32;
  if (i == m - 1 || (key[i + 1] >> 32) != g) width[g] = 32 * (C[i] - first[g] + 1);
}

__global__ void index_kernel(const unsigned long long* key, const uint32_t* val, const long long* C, long long m,
                             const long long* first, const uint32_t* pos, const long long* groupOff, uint32_t base,
                             uint32_t* idx) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long g = key[i] >> 32;
  const uint32_t e = val[i];
  idx[groupOff[g] + 32 * (C[i] - first[g]) + (pos[e] & 31)] = base + e;
}

// out[t] = init[t] (or 0) + t's partials of one list summed in slot order,
// one thread per target, R right-hand sides per entry.
template <int R>
__global__ void seg_sum_kernel(const double* __restrict__ part, const uint32_t* __restrict__ idx,
                               const long long* __restrict__ groupOff, const double* __restrict__ init,
                               double* __restrict__ zp, int n, int lo, int hi, int nrhs) {
  const long long t = lo + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= hi) return;
  const long long g = t >> 5, w = (groupOff[g + 1] - groupOff[g]) / 32;
  const uint32_t* col = idx + groupOff[g] + (t & 31);
  constexpr int RR = R > 0 ? R : 1;
  for (int r0 = 0; r0 < nrhs; r0 += RR) {
    double acc[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) acc[r] = init ? init[static_cast<size_t>(r0 + r) * n + t] : 0.0;
    // pads index the all-zero row past the last entry (x + 0 == x): no
    // branch, so the unrolled loads of several slots are in flight together
#pragma unroll 8
    for (long long j = 0; j < w; ++j) {
      const uint32_t e = col[32 * j];
      const double* p = part + static_cast<size_t>(e) * nrhs + r0;
      if constexpr (RR % 2 == 0) {
#pragma unroll
        for (int r = 0; r < RR; r += 2) {
          const double2 v = *reinterpret_cast<const double2*>(p + r);
          acc[r] += v.x;
          acc[r + 1] += v.y;
        }
      } else {
        acc[0] += p[0];
      }
    }
#pragma unroll
    for (int r = 0; r < RR; ++r) zp[static_cast<size_t>(r0 + r) * n + t] = acc[r];
  }
}

// moments[rhs][node][c] = sum over the node's S2M tiles [t0, t1), in tile
// order, of the per-tile partials part[tile][rhs][c].
__global__ void tile_sum_kernel(const double* __restrict__ part, const int* __restrict__ ranges, int PC, int nrhs,
                                int nodes, double* __restrict__ moments) {
  const int node = ranges[3 * blockIdx.x], t0 = ranges[3 * blockIdx.x + 1], t1 = ranges[3 * blockIdx.x + 2];
  for (int i = threadIdx.x; i < PC * nrhs; i += blockDim.x) {
    const int rhs = i / PC, c = i - rhs * PC;
    double acc = 0.0;
    for (int t = t0; t < t1; ++t) acc += part[(static_cast<size_t>(t) * nrhs + rhs) * PC + c];
    moments[(static_cast<size_t>(rhs) * nodes + node) * PC + c] = acc;
  }
}

template <class K, class V>
void cubSortPairs(const K* keysIn, K* keysOut, const V* valsIn, V* valsOut, long long m, int bits, cudaStream_t st) {
  size_t bytes = 0;
  FKTB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keysIn, keysOut, valsIn, valsOut, m, 0, bits, st));
  DeviceBuffer<unsigned char> temp(bytes + 1);
  FKTB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), bytes, keysIn, keysOut, valsIn, valsOut, m, 0, bits, st));
  FKTB_CUDA(cudaStreamSynchronize(st));  // temp is released on return
}

template <class In, class Out>
void cubExclusiveScan(const In* in, Out* out, int n, cudaStream_t st) {
  // out[0] = 0, out[i + 1] = in[0] + ... + in[i]
  FKTB_CUDA(cudaMemsetAsync(out, 0, sizeof(Out), st));
  size_t bytes = 0;
  FKTB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, n, st));
  DeviceBuffer<unsigned char> temp(bytes + 1);
  FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, in, out + 1, n, st));
  FKTB_CUDA(cudaStreamSynchronize(st));
}

int grid(long long m, int threads) { return static_cast<int>((m + threads - 1) / threads); }

}  // namespace

void buildDeterministic(DevicePlan& plan) {
  const DeviceTree& t = *plan.tree;
  cudaStream_t st = plan.stream;
  const int n = t.n;
  const long long nm = t.nearTotal, fm = t.farTotal;
  if (nm + fm + 1 >= static_cast<long long>(std::numeric_limits<uint32_t>::max()))
    throw std::invalid_argument("unsupported on the GPU path: deterministic mode needs < 2^32 near + far entries");
  plan.slotsTotal = nm + fm;
  const int groups = (n + 31) / 32;
  // one sliced index per list (near: entries [0, nm) of the partials, far: [nm, nm + fm))
  int nbits = 1;
  while ((1 << nbits) < t.nodes) ++nbits;
  int gbits = 1;
  while ((1ll << gbits) < groups) ++gbits;
  auto indexOf = [&](const long long* off, const uint32_t* pos, long long m, uint32_t base, DetIndex& out) {
    out.groupOff.resize(static_cast<size_t>(groups) + 1);
    DeviceBuffer<long long> width(static_cast<size_t>(groups));
    FKTB_CUDA(cudaMemsetAsync(width.get(), 0, width.bytes(), st));
    if (m == 0) {
      cubExclusiveScan(width.get(), out.groupOff.get(), groups, st);
      out.idx.resize(1);
      return;
    }
    DeviceBuffer<unsigned long long> key(static_cast<size_t>(m)), keyOut(static_cast<size_t>(m));
    DeviceBuffer<uint32_t> vals(static_cast<size_t>(m)), valsOut(static_cast<size_t>(m));
    entry_key_kernel<<<t.nodes, 256, 0, st>>>(off, pos, key.get());
    iota_kernel<<<grid(m, 256), 256, 0, st>>>(vals.get(), m);
    FKTB_CUDA(cudaGetLastError());
    // stable: entries of one (group, node) stay ascending (= ascending targets)
    cubSortPairs(key.get(), keyOut.get(), vals.get(), valsOut.get(), m, 32 + gbits, st);
    key.release();
    vals.release();
    DeviceBuffer<long long> flag(static_cast<size_t>(m)), C(static_cast<size_t>(m)), first(static_cast<size_t>(groups));
    new_slot_kernel<<<grid(m, 256), 256, 0, st>>>(keyOut.get(), m, flag.get());
    FKTB_CUDA(cudaGetLastError());
    {
      size_t bytes = 0;
      FKTB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, flag.get(), C.get(), m, st));
      DeviceBuffer<unsigned char> temp(bytes + 1);
      FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, flag.get(), C.get(), m, st));
      FKTB_CUDA(cudaStreamSynchronize(st));
    }
    group_first_kernel<<<grid(m, 256), 256, 0, st>>>(keyOut.get(), C.get(), m, first.get());
    group_width_kernel<<<grid(m, 256), 256, 0, st>>>(keyOut.get(), C.get(), m, first.get(), width.get());
    FKTB_CUDA(cudaGetLastError());
    cubExclusiveScan(width.get(), out.groupOff.get(), groups, st);
    long long slots = 0;
    FKTB_CUDA(cudaMemcpy(&slots, out.groupOff.get() + groups, sizeof(long long), cudaMemcpyDeviceToHost));
    out.idx.resize(std::max<long long>(1, slots));
    fill_kernel<<<grid(static_cast<long long>(out.idx.size()), 256), 256, 0, st>>>(
        out.idx.get(), static_cast<long long>(out.idx.size()), static_cast<uint32_t>(nm + fm));  // pads: the zero row
    index_kernel<<<grid(m, 256), 256, 0, st>>>(keyOut.get(), valsOut.get(), C.get(), m, first.get(), pos,
                                               out.groupOff.get(), base, out.idx.get());
    FKTB_CUDA(cudaGetLastError());
    FKTB_CUDA(cudaStreamSynchronize(st));
  };
  (void)nbits;
  indexOf(t.dNearOff.get(), t.dNearPos.get(), nm, 0, plan.detNear);
  indexOf(t.dFarOff.get(), t.dFarPos.get(), fm, static_cast<uint32_t>(nm), plan.detFar);
  plan.detBuilt = true;
}

// S2M tiles grouped by node (tiles of a node are consecutive in s2mTilesHost).
void buildDetTileRanges(DevicePlan& plan) {
  std::vector<int> ranges;
  const auto& tl = plan.s2mTilesHost;
  for (size_t i = 0; i < tl.size();) {
    size_t j = i;
    while (j < tl.size() && tl[j].node == tl[i].node) ++j;
    ranges.insert(ranges.end(), {tl[i].node, static_cast<int>(i), static_cast<int>(j)});
    i = j;
  }
  plan.detTileNodes = static_cast<int>(ranges.size() / 3);
  plan.dDetTileRanges.resize(std::max<size_t>(1, ranges.size()));
  if (!ranges.empty())
    FKTB_CUDA(cudaMemcpy(plan.dDetTileRanges.get(), ranges.data(), ranges.size() * sizeof(int), cudaMemcpyHostToDevice));
}

ZOut zoutFor(const DevicePlan& plan, double* zp, int nrhs, bool far) {
  ZOut o{zp, nullptr, nrhs, 0, plan.n};
  if (plan.options.deterministic) {
    o.part = plan.dPart.get();
    o.base = far ? plan.tree->nearTotal : 0;
  }
  return o;
}

ZOut zoutShift(ZOut o, int r0) {
  o.zp += static_cast<size_t>(r0) * o.n;
  if (o.part) o.part += r0;
  return o;
}

// far: z_far = the far partials (side stream, after the M2T); near: z =
// z_far + the near partials (after the join).
void launchDetReduce(const DevicePlan& plan, double* zp, int nrhs, bool far, cudaStream_t st) {
  const int lo = static_cast<int>(plan.shardLo), hi = static_cast<int>(plan.shardHi);
  if (hi <= lo) return;
  const int blocks = grid(hi - lo, 256);
  const double* part = plan.dPart.get();
  const DetIndex& ix = far ? plan.detFar : plan.detNear;
  const uint32_t* idx = ix.idx.get();
  const long long* off = ix.groupOff.get();
  const double* init = far ? nullptr : plan.dZf.get();
  double* out = far ? plan.dZf.get() : zp;
  if (nrhs % 16 == 0)
    seg_sum_kernel<16><<<blocks, 256, 0, st>>>(part, idx, off, init, out, plan.n, lo, hi, nrhs);
  else if (nrhs % 8 == 0)
    seg_sum_kernel<8><<<blocks, 256, 0, st>>>(part, idx, off, init, out, plan.n, lo, hi, nrhs);
  else if (nrhs % 4 == 0)
    seg_sum_kernel<4><<<blocks, 256, 0, st>>>(part, idx, off, init, out, plan.n, lo, hi, nrhs);
  else if (nrhs % 2 == 0)
    seg_sum_kernel<2><<<blocks, 256, 0, st>>>(part, idx, off, init, out, plan.n, lo, hi, nrhs);
  else
    seg_sum_kernel<1><<<blocks, 256, 0, st>>>(part, idx, off, init, out, plan.n, lo, hi, nrhs);
  FKTB_CUDA(cudaGetLastError());
}

void launchDetTileSum(const DevicePlan& plan, const double* part, int PC, int nrhs, double* moments, cudaStream_t st) {
  if (plan.detTileNodes == 0) return;
  tile_sum_kernel<<<plan.detTileNodes, 128, 0, st>>>(part, plan.dDetTileRanges.get(), PC, nrhs, plan.tree->nodes,
                                                     moments);
  FKTB_CUDA(cudaGetLastError());
}

}  // namespace fktb
