// K1 (partition tree) and K2 (point-wise interaction sets) on the GPU.
//
// K1 restates proj/src/tree.cpp:13-171 level-synchronously: one CTA per node
// being split at the current depth computes the tight box, the aspect
// regularisation, center and radius, the longest-side axis, the clamped upper
// median (exact k-th smallest by an 8-pass MSD radix select on order-preserving
// 64-bit keys) and the stable `<=` partition (ballot/popc scan), including the
// fallback split at the largest value below the maximum. Node numbering is
// converted from BFS to the reference's pre-order on the host.
//
// K2 restates tree.cpp:173-213 per target: each thread walks the tree from the
// root, emitting (node, position) for far nodes and (leaf, position) for the
// near leaf; a stable radix sort by node gives the node-major CSR with targets
// ascending.
//
// All floating-point here must be bit-identical to the reference:
// this file is compiled with -fmad=false (no contraction) and uses only
// IEEE-exact operations (+ - * / sqrt, min/max, compares).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <numeric>

#include "plan.hpp"

namespace fktb {
namespace {

constexpr int kTreeThreads = 512;

__device__ __forceinline__ unsigned long long toKey(double x) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double fromKey(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}

struct LevelArgs {
  int n, d, leafCap;
  double* pc;
  double* tc;
  uint32_t* order;
  uint32_t* torder;
  const int* segB;
  const int* segE;
  double* outLo;
  double* outHi;
  double* outCenter;
  double* outRadius;
  int* outMid;  // -1 for a leaf
};

__global__ void __launch_bounds__(kTreeThreads) tree_level_kernel(LevelArgs A) {
  const int s = blockIdx.x;
  const int b = A.segB[s], e = A.segE[s];
  const int cnt = e - b;
  const int n = A.n, d = A.d;
  const int tid = threadIdx.x, bdim = blockDim.x;
  __shared__ double red[32];
  __shared__ long long redll[32];
  __shared__ double lo[FKTB_MAX_DIM], hi[FKTB_MAX_DIM], ctr[FKTB_MAX_DIM];
  __shared__ double sExtent;
  __shared__ unsigned hist[256];
  __shared__ unsigned long long sPrefix;
  __shared__ int sK;
  __shared__ int sAxis;
  __shared__ double sClampLo, sClampHi;
  __shared__ int warpCnt[kTreeThreads / 32];

  // Tight box (tree.cpp:48-56).
  for (int a = 0; a < d; ++a) {
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
    const double* col = A.pc + static_cast<size_t>(a) * n;
    for (int pos = b + tid; pos < e; pos += bdim) {
      const double v = col[pos];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    mn = block_reduce<1>(mn, red);
    mx = block_reduce<2>(mx, red);
    if (tid == 0) {
      lo[a] = mn;
      hi[a] = mx;
    }
  }
  __syncthreads();
  if (tid == 0) {
    double extent = 0.0;
    for (int a = 0; a < d; ++a) extent = extent + (hi[a] - lo[a]);
    // regularizeBox (tree.cpp:13-25)
    double maxSide = 0.0;
    for (int a = 0; a < d; ++a) {
      const double side = hi[a] - lo[a];
      maxSide = maxSide < side ? side : maxSide;
    }
    if (maxSide > 0.0) {
      for (int a = 0; a < d; ++a) {
        const double side = hi[a] - lo[a];
        if (side < 0.5 * maxSide) {
          const double pad = 0.5 * (0.5 * maxSide - side);
          lo[a] = lo[a] - pad;
          hi[a] = hi[a] + pad;
        }
      }
    }
    for (int a = 0; a < d; ++a) ctr[a] = 0.5 * (lo[a] + hi[a]);
    sExtent = extent;
  }
  __syncthreads();
  // Radius (tree.cpp:64-74): sequential per-axis sum, exact max.
  double r2 = 0.0;
  for (int pos = b + tid; pos < e; pos += bdim) {
    double dist2 = 0.0;
    for (int a = 0; a < d; ++a) {
      const double t = A.pc[static_cast<size_t>(a) * n + pos] - ctr[a];
      dist2 = dist2 + t * t;
    }
    r2 = fmax(r2, dist2);
  }
  r2 = block_reduce<2>(r2, red);
  if (tid == 0) {
    for (int a = 0; a < d; ++a) {
      A.outLo[static_cast<size_t>(s) * d + a] = lo[a];
      A.outHi[static_cast<size_t>(s) * d + a] = hi[a];
      A.outCenter[static_cast<size_t>(s) * d + a] = ctr[a];
    }
    A.outRadius[s] = sqrt(r2);
  }
  if (cnt <= A.leafCap || sExtent == 0.0) {
    if (tid == 0) A.outMid[s] = -1;
    return;
  }

  // Axis and clamp interval (tree.cpp:81-115).
  if (tid == 0) {
    int axis = 0;
    double bestSide = -1.0;
    for (int a = 0; a < d; ++a) {
      const double side = hi[a] - lo[a];
      if (side > bestSide) {
        bestSide = side;
        axis = a;
      }
    }
    const double l = lo[axis], h = hi[axis];
    double maxOther = 0.0, minOther = __longlong_as_double(0x7ff0000000000000ll);
    for (int a = 0; a < d; ++a) {
      if (a == axis) continue;
      const double side = hi[a] - lo[a];
      maxOther = maxOther < side ? side : maxOther;
      minOther = side < minOther ? side : minOther;
    }
    double cl = l, ch = h;
    if (d > 1) {
      const double c1 = l + 0.5 * maxOther, c2 = h - 2.0 * minOther;
      cl = c1 < c2 ? c2 : c1;
      const double c3 = l + 2.0 * minOther, c4 = h - 0.5 * maxOther;
      ch = c4 < c3 ? c4 : c3;
      if (cl > ch) cl = ch = 0.5 * (l + h);
    }
    sAxis = axis;
    sClampLo = cl;
    sClampHi = ch;
    sPrefix = 0ull;
    sK = cnt / 2;
  }
  __syncthreads();
  const int axis = sAxis;
  const double* col = A.pc + static_cast<size_t>(axis) * n;

  // Exact (cnt/2)-th smallest value: MSD radix select, 8 bits per pass
  // (equivalent to std::nth_element's values[size/2], tree.cpp:116-119).
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    const unsigned long long highMask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    for (int i = tid; i < 256; i += bdim) hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sPrefix;
    for (int pos = b + tid; pos < e; pos += bdim) {
      const unsigned long long key = toKey(col[pos]);
      if ((key & highMask) == prefix) {
        const unsigned dig = static_cast<unsigned>((key >> shift) & 255ull);
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, dig);
        if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&hist[dig], __popc(peers));
      }
    }
    __syncthreads();
    if (tid == 0) {
      int k = sK;
      unsigned cum = 0;
      for (int dg = 0; dg < 256; ++dg) {
        if (cum + hist[dg] > static_cast<unsigned>(k)) {
          sPrefix = prefix | (static_cast<unsigned long long>(dg) << shift);
          sK = k - static_cast<int>(cum);
          break;
        }
        cum += hist[dg];
      }
    }
    __syncthreads();
  }
  double split;
  {
    const double v = fromKey(sPrefix);
    const double cl = sClampLo, ch = sClampHi;
    split = v < cl ? cl : (ch < v ? ch : v);  // std::clamp
  }

  // Lower count; fallback split at the largest value below the maximum
  // (tree.cpp:136-159).
  long long lower = 0;
  for (int pos = b + tid; pos < e; pos += bdim) lower += col[pos] <= split ? 1 : 0;
  lower = block_sum_ll(lower, redll);
  if (lower == 0 || lower == cnt) {
    double mx = -__longlong_as_double(0x7ff0000000000000ll);
    for (int pos = b + tid; pos < e; pos += bdim) mx = fmax(mx, col[pos]);
    mx = block_reduce<2>(mx, red);
    double below = -__longlong_as_double(0x7ff0000000000000ll);
    for (int pos = b + tid; pos < e; pos += bdim) {
      const double v = col[pos];
      if (v < mx) below = fmax(below, v);
    }
    below = block_reduce<2>(below, red);
    split = below;
    lower = 0;
    for (int pos = b + tid; pos < e; pos += bdim) lower += col[pos] <= split ? 1 : 0;
    lower = block_sum_ll(lower, redll);
  }

  // Stable partition into the scratch arrays, then copy back.
  const int L = static_cast<int>(lower);
  const int lane = tid & 31, warp = tid >> 5, nw = bdim >> 5;
  int lowerBase = 0, upperBase = 0;
  for (int start = b; start < e; start += bdim) {
    const int pos = start + tid;
    const bool valid = pos < e;
    const bool flag = valid && col[pos] <= split;
    const unsigned ballot = __ballot_sync(0xffffffffu, flag);
    const int rank = __popc(ballot & ((1u << lane) - 1u));
    if (lane == 0) warpCnt[warp] = __popc(ballot);
    __syncthreads();
    int wpre = 0, chunkLower = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < warp) wpre += warpCnt[w];
      chunkLower += warpCnt[w];
    }
    if (valid) {
      const int before = wpre + rank;
      const int dst = flag ? b + lowerBase + before : b + L + upperBase + (pos - start - before);
      for (int a = 0; a < d; ++a) A.tc[static_cast<size_t>(a) * n + dst] = A.pc[static_cast<size_t>(a) * n + pos];
      A.torder[dst] = A.order[pos];
    }
    const int chunk = min(bdim, e - start);
    lowerBase += chunkLower;
    upperBase += chunk - chunkLower;
    __syncthreads();
  }
  __syncthreads();
  for (int pos = b + tid; pos < e; pos += bdim) {
    for (int a = 0; a < d; ++a) A.pc[static_cast<size_t>(a) * n + pos] = A.tc[static_cast<size_t>(a) * n + pos];
    A.order[pos] = A.torder[pos];
  }
  if (tid == 0) A.outMid[s] = b + L;
}

__global__ void transpose_to_soa(const double* x, int n, int d, double* pc, uint32_t* order) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int a = 0; a < d; ++a) pc[static_cast<size_t>(a) * n + i] = x[static_cast<size_t>(i) * d + a];
  order[i] = static_cast<uint32_t>(i);
}

// ---------------------------------------------------------------------------
// K2: per-target traversal. MODE 0 counts, MODE 1 writes (node, pos) pairs.
struct SetsArgs {
  int n, d, nodes;
  const double* pc;
  const double* center;
  const double* limit2;
  const int* left;
  const int* right;
  int* farCnt;
  int* nearCnt;
  const long long* farStart;
  const long long* nearStart;
  uint32_t* farNode;
  uint32_t* farPos;
  uint32_t* nearNode;
  uint32_t* nearPos;
};

template <int MODE>
__global__ void sets_kernel(SetsArgs A) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= A.n) return;
  double pt[FKTB_MAX_DIM];
  for (int a = 0; a < A.d; ++a) pt[a] = A.pc[static_cast<size_t>(a) * A.n + pos];
  int stack[128];
  int sp = 0;
  stack[sp++] = 0;
  int nf = 0, nn = 0;
  long long fo = MODE ? A.farStart[pos] : 0, no = MODE ? A.nearStart[pos] : 0;
  while (sp > 0) {
    const int b = stack[--sp];
    double dist2 = 0.0;
    const double* c = A.center + static_cast<size_t>(b) * A.d;
    for (int a = 0; a < A.d; ++a) {
      const double t = pt[a] - c[a];
      dist2 = dist2 + t * t;
    }
    if (dist2 > A.limit2[b]) {
      if (MODE) {
        A.farNode[fo] = static_cast<uint32_t>(b);
        A.farPos[fo] = static_cast<uint32_t>(pos);
        ++fo;
      }
      ++nf;
    } else if (A.left[b] < 0) {
      if (MODE) {
        A.nearNode[no] = static_cast<uint32_t>(b);
        A.nearPos[no] = static_cast<uint32_t>(pos);
        ++no;
      }
      ++nn;
    } else {
      stack[sp++] = A.right[b];
      stack[sp++] = A.left[b];
    }
  }
  if (!MODE) {
    A.farCnt[pos] = nf;
    A.nearCnt[pos] = nn;
  }
}

__global__ void csr_offsets(const uint32_t* keys, long long total, int nodes, long long* off) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nodes) return;
  long long lo = 0, hi = total;  // first index with key >= b
  while (lo < hi) {
    const long long mid = (lo + hi) / 2;
    if (keys[mid] < static_cast<uint32_t>(b))
      lo = mid + 1;
    else
      hi = mid;
  }
  off[b] = lo;
}

int bitsFor(int v) {
  int b = 1;
  while ((1ll << b) <= v) ++b;
  return b;
}

void sortPairsToCsr(DeviceBuffer<uint32_t>& keys, DeviceBuffer<uint32_t>& vals, long long total, int nodes,
                    DeviceBuffer<long long>& dOff, std::vector<long long>& hOff, DeviceBuffer<uint32_t>& outPos,
                    cudaStream_t st) {
  dOff.resize(static_cast<size_t>(nodes) + 1);
  outPos.resize(static_cast<size_t>(std::max<long long>(total, 1)));
  hOff.assign(static_cast<size_t>(nodes) + 1, 0);
  if (total == 0) {
    FKTB_CUDA(cudaMemsetAsync(dOff.get(), 0, dOff.bytes(), st));
    return;
  }
  DeviceBuffer<uint32_t> keysOut(static_cast<size_t>(total));
  size_t tempBytes = 0;
  FKTB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tempBytes, keys.get(), keysOut.get(), vals.get(), outPos.get(),
                                            static_cast<int64_t>(total), 0, bitsFor(nodes), st));
  DeviceBuffer<unsigned char> temp(tempBytes);
  FKTB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tempBytes, keys.get(), keysOut.get(), vals.get(),
                                            outPos.get(), static_cast<int64_t>(total), 0, bitsFor(nodes), st));
  csr_offsets<<<(nodes + 1 + 255) / 256, 256, 0, st>>>(keysOut.get(), total, nodes, dOff.get());
  FKTB_CUDA(cudaGetLastError());
  FKTB_CUDA(cudaMemcpyAsync(hOff.data(), dOff.get(), dOff.bytes(), cudaMemcpyDeviceToHost, st));
  FKTB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void buildTreeGpu(DeviceTree& t, const double* hostX, int n, int d, int leafCapacity, cudaStream_t st) {
  if (leafCapacity < 1) throw std::invalid_argument("leaf capacity must be >= 1");
  if (n < 1) throw std::invalid_argument("point cloud must be nonempty");
  if (d < 1 || d > FKTB_MAX_DIM) throw std::invalid_argument("GPU tree supports 1 <= d <= 16");
  t.n = n;
  t.d = d;
  t.leafCapacity = leafCapacity;
  t.stream = st;
  const size_t nd = static_cast<size_t>(n) * d;
  DeviceBuffer<double> x(nd), tc(nd);
  DeviceBuffer<uint32_t> torder(static_cast<size_t>(n));
  t.pc.resize(nd);
  t.order.resize(static_cast<size_t>(n));
  FKTB_CUDA(cudaMemcpyAsync(x.get(), hostX, nd * sizeof(double), cudaMemcpyHostToDevice, st));
  transpose_to_soa<<<(n + 255) / 256, 256, 0, st>>>(x.get(), n, d, t.pc.get(), t.order.get());
  FKTB_CUDA(cudaGetLastError());

  // BFS-ordered node records.
  struct Rec {
    int begin, end, left = -1, right = -1, depth = 0;
    std::vector<double> lo, hi, c;
    double radius = 0.0;
  };
  std::vector<Rec> recs;
  recs.push_back(Rec{0, n});
  std::vector<int> level = {0};
  const int maxSeg = std::max(1, 2 * (n / leafCapacity + 1) + 2);
  DeviceBuffer<int> dSegB(static_cast<size_t>(maxSeg)), dSegE(static_cast<size_t>(maxSeg)), dMid(static_cast<size_t>(maxSeg));
  DeviceBuffer<double> dLo(static_cast<size_t>(maxSeg) * d), dHi(static_cast<size_t>(maxSeg) * d),
      dC(static_cast<size_t>(maxSeg) * d), dR(static_cast<size_t>(maxSeg));
  std::vector<int> hb, he, hmid;
  std::vector<double> hlo, hhi, hc, hr;
  int depth = 0;
  while (!level.empty()) {
    const int ns = static_cast<int>(level.size());
    if (ns > maxSeg) throw std::runtime_error("tree build: segment buffer overflow");
    hb.resize(ns);
    he.resize(ns);
    for (int i = 0; i < ns; ++i) {
      hb[i] = recs[static_cast<size_t>(level[i])].begin;
      he[i] = recs[static_cast<size_t>(level[i])].end;
    }
    FKTB_CUDA(cudaMemcpyAsync(dSegB.get(), hb.data(), ns * sizeof(int), cudaMemcpyHostToDevice, st));
    FKTB_CUDA(cudaMemcpyAsync(dSegE.get(), he.data(), ns * sizeof(int), cudaMemcpyHostToDevice, st));
    LevelArgs A{n,        d,        leafCapacity, t.pc.get(), tc.get(), t.order.get(), torder.get(), dSegB.get(),
                dSegE.get(), dLo.get(), dHi.get(),   dC.get(),   dR.get(),  dMid.get()};
    tree_level_kernel<<<ns, kTreeThreads, 0, st>>>(A);
    FKTB_CUDA(cudaGetLastError());
    hmid.resize(ns);
    hlo.resize(static_cast<size_t>(ns) * d);
    hhi.resize(static_cast<size_t>(ns) * d);
    hc.resize(static_cast<size_t>(ns) * d);
    hr.resize(ns);
    FKTB_CUDA(cudaMemcpyAsync(hmid.data(), dMid.get(), ns * sizeof(int), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaMemcpyAsync(hlo.data(), dLo.get(), hlo.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaMemcpyAsync(hhi.data(), dHi.get(), hhi.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaMemcpyAsync(hc.data(), dC.get(), hc.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaMemcpyAsync(hr.data(), dR.get(), hr.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaStreamSynchronize(st));
    std::vector<int> next;
    for (int i = 0; i < ns; ++i) {
      const int id = level[i];
      {
        Rec& r = recs[static_cast<size_t>(id)];
        r.lo.assign(hlo.begin() + static_cast<long>(i) * d, hlo.begin() + static_cast<long>(i + 1) * d);
        r.hi.assign(hhi.begin() + static_cast<long>(i) * d, hhi.begin() + static_cast<long>(i + 1) * d);
        r.c.assign(hc.begin() + static_cast<long>(i) * d, hc.begin() + static_cast<long>(i + 1) * d);
        r.radius = hr[i];
      }
      if (hmid[i] >= 0) {
        const int b = recs[static_cast<size_t>(id)].begin, e = recs[static_cast<size_t>(id)].end;
        const int lid = static_cast<int>(recs.size());
        recs.push_back(Rec{b, hmid[i]});
        recs.back().depth = depth + 1;
        recs.push_back(Rec{hmid[i], e});
        recs.back().depth = depth + 1;
        recs[static_cast<size_t>(id)].left = lid;
        recs[static_cast<size_t>(id)].right = lid + 1;
        next.push_back(lid);
        next.push_back(lid + 1);
      }
    }
    level.swap(next);
    if (!level.empty()) ++depth;
  }
  t.depth = depth;

  // BFS -> pre-order (left subtree first), tree.cpp:166-169.
  const int nodes = static_cast<int>(recs.size());
  std::vector<int> pre(static_cast<size_t>(nodes));
  {
    std::vector<int> stack = {0};
    int next = 0;
    while (!stack.empty()) {
      const int id = stack.back();
      stack.pop_back();
      pre[static_cast<size_t>(id)] = next++;
      if (recs[static_cast<size_t>(id)].left >= 0) {
        stack.push_back(recs[static_cast<size_t>(id)].right);
        stack.push_back(recs[static_cast<size_t>(id)].left);
      }
    }
  }
  t.nodes = nodes;
  t.begin.assign(static_cast<size_t>(nodes), 0);
  t.end.assign(static_cast<size_t>(nodes), 0);
  t.left.assign(static_cast<size_t>(nodes), -1);
  t.right.assign(static_cast<size_t>(nodes), -1);
  t.boxLo.assign(static_cast<size_t>(nodes) * d, 0.0);
  t.boxHi.assign(static_cast<size_t>(nodes) * d, 0.0);
  t.center.assign(static_cast<size_t>(nodes) * d, 0.0);
  t.radius.assign(static_cast<size_t>(nodes), 0.0);
  for (int id = 0; id < nodes; ++id) {
    const Rec& r = recs[static_cast<size_t>(id)];
    const size_t p = static_cast<size_t>(pre[static_cast<size_t>(id)]);
    t.begin[p] = static_cast<uint32_t>(r.begin);
    t.end[p] = static_cast<uint32_t>(r.end);
    t.left[p] = r.left >= 0 ? pre[static_cast<size_t>(r.left)] : -1;
    t.right[p] = r.right >= 0 ? pre[static_cast<size_t>(r.right)] : -1;
    for (int a = 0; a < d; ++a) {
      t.boxLo[p * d + a] = r.lo[static_cast<size_t>(a)];
      t.boxHi[p * d + a] = r.hi[static_cast<size_t>(a)];
      t.center[p * d + a] = r.c[static_cast<size_t>(a)];
    }
    t.radius[p] = r.radius;
  }
  t.dCenter.resize(t.center.size());
  t.dLeft.resize(static_cast<size_t>(nodes));
  t.dRight.resize(static_cast<size_t>(nodes));
  t.dBegin.resize(static_cast<size_t>(nodes));
  t.dEnd.resize(static_cast<size_t>(nodes));
  FKTB_CUDA(cudaMemcpyAsync(t.dCenter.get(), t.center.data(), t.dCenter.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(t.dLeft.get(), t.left.data(), t.dLeft.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(t.dRight.get(), t.right.data(), t.dRight.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(t.dBegin.get(), t.begin.data(), t.dBegin.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaMemcpyAsync(t.dEnd.get(), t.end.data(), t.dEnd.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaStreamSynchronize(st));
}

void computeSetsGpu(DeviceTree& t, double theta) {
  if (!(theta > 0.0 && theta < 1.0)) throw std::invalid_argument("theta must be in (0, 1)");
  cudaStream_t st = t.stream;
  t.theta = theta;
  const int n = t.n, nodes = t.nodes;
  // limit2 exactly as tree.cpp:191-192.
  std::vector<double> lim2(static_cast<size_t>(nodes));
  for (int b = 0; b < nodes; ++b) {
    volatile double limit = t.radius[static_cast<size_t>(b)] / theta;
    lim2[static_cast<size_t>(b)] = limit * limit;
  }
  t.dLimit2.resize(static_cast<size_t>(nodes));
  FKTB_CUDA(cudaMemcpyAsync(t.dLimit2.get(), lim2.data(), t.dLimit2.bytes(), cudaMemcpyHostToDevice, st));

  DeviceBuffer<int> farCnt(static_cast<size_t>(n)), nearCnt(static_cast<size_t>(n));
  DeviceBuffer<long long> farStart(static_cast<size_t>(n) + 1), nearStart(static_cast<size_t>(n) + 1);
  SetsArgs A{n, t.d, nodes, t.pc.get(), t.dCenter.get(), t.dLimit2.get(), t.dLeft.get(), t.dRight.get(),
             farCnt.get(), nearCnt.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const int blocks = (n + 127) / 128;
  sets_kernel<0><<<blocks, 128, 0, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
  // Exclusive scans of the per-target counts (int -> int64).
  {
    FKTB_CUDA(cudaMemsetAsync(farStart.get(), 0, sizeof(long long), st));
    FKTB_CUDA(cudaMemsetAsync(nearStart.get(), 0, sizeof(long long), st));
    size_t bytes = 0;
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, farCnt.get(), farStart.get() + 1, n, st));
    DeviceBuffer<unsigned char> temp(bytes);
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, farCnt.get(), farStart.get() + 1, n, st));
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, nearCnt.get(), nearStart.get() + 1, n, st));
  }
  long long totals[2] = {0, 0};
  FKTB_CUDA(cudaMemcpyAsync(&totals[0], farStart.get() + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FKTB_CUDA(cudaMemcpyAsync(&totals[1], nearStart.get() + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FKTB_CUDA(cudaStreamSynchronize(st));
  t.farTotal = totals[0];
  t.nearTotal = totals[1];
  DeviceBuffer<uint32_t> farNode(static_cast<size_t>(std::max(1ll, t.farTotal))), farPos(static_cast<size_t>(std::max(1ll, t.farTotal)));
  DeviceBuffer<uint32_t> nearNode(static_cast<size_t>(std::max(1ll, t.nearTotal))), nearPos(static_cast<size_t>(std::max(1ll, t.nearTotal)));
  A.farStart = farStart.get();
  A.nearStart = nearStart.get();
  A.farNode = farNode.get();
  A.farPos = farPos.get();
  A.nearNode = nearNode.get();
  A.nearPos = nearPos.get();
  sets_kernel<1><<<blocks, 128, 0, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
  farCnt.release();
  nearCnt.release();
  farStart.release();
  nearStart.release();
  sortPairsToCsr(farNode, farPos, t.farTotal, nodes, t.dFarOff, t.farOff, t.dFarPos, st);
  sortPairsToCsr(nearNode, nearPos, t.nearTotal, nodes, t.dNearOff, t.nearOff, t.dNearPos, st);
  t.hasSets = true;
}

void materializeSets(const DeviceTree& t, bool far, std::vector<long long>& off, std::vector<uint32_t>& idx) {
  const long long total = far ? t.farTotal : t.nearTotal;
  off = far ? t.farOff : t.nearOff;
  idx.assign(static_cast<size_t>(total), 0);
  std::vector<uint32_t> order(static_cast<size_t>(t.n));
  FKTB_CUDA(cudaMemcpy(order.data(), t.order.get(), order.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (total > 0)
    FKTB_CUDA(cudaMemcpy(idx.data(), far ? t.dFarPos.get() : t.dNearPos.get(), static_cast<size_t>(total) * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost));
  for (auto& v : idx) v = order[v];
  for (int b = 0; b < t.nodes; ++b)
    std::sort(idx.begin() + off[static_cast<size_t>(b)], idx.begin() + off[static_cast<size_t>(b) + 1]);
}

}  // namespace fktb
