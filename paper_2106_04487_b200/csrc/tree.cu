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
  const int* outIdx;  // level slot of segment blockIdx.x (nullptr: the same)
  double* outLo;
  double* outHi;
  double* outCenter;
  double* outRadius;
  int* outMid;  // -1 for a leaf
};

__global__ void __launch_bounds__(kTreeThreads) tree_level_kernel(LevelArgs A) {
  const int s = A.outIdx ? A.outIdx[blockIdx.x] : static_cast<int>(blockIdx.x);
  const int b = A.segB[blockIdx.x], e = A.segE[blockIdx.x];
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

// ---------------------------------------------------------------------------
// Wide levels: the top of the tree has few segments with many points each, so
// one CTA per segment leaves most of the 148 SMs idle (cfg2: the root level
// alone took 12.6 ms, the top four 24 ms of 26). There every phase of the
// split runs over work items of kWideItem points with one CTA each; the
// segment-wide results are combined by exact, order-independent atomics
// (min / max on order-preserving keys, integer counts), so the tree stays
// bit-identical to the reference:
//   box -> finalize (regularize, centre) -> radius -> finalize (leaf? axis,
//   clamp) -> 8 x (histogram, select) -> split, lower counts [-> fallback
//   max, below, recount] -> per-item prefix -> stable partition -> copy back.
constexpr int kWideItem = 8192;     // points per work item
constexpr int kWideThreads = 256;
constexpr int kWideMin = 2 * kWideItem;  // segments above this size take the wide path

struct WideSeg {
  unsigned long long boxKey[FKTB_MAX_DIM][2];  // min, max keys per axis
  unsigned long long r2Key;                    // max squared distance (bits)
  unsigned long long prefix;                   // radix-select prefix
  unsigned long long mxKey, belowKey;          // fallback split
  unsigned long long lower;                    // points <= split
  double ctr[FKTB_MAX_DIM];
  double split, clampLo, clampHi, extent;
  int k, axis, active, fallback, begin, end;
  unsigned hist[256];
};

struct WideArgs {
  int n, d, leafCap, ns, items;
  const int* outIdx;   // level slot of wide segment j
  const int* segItem;  // items of wide segment j: [segItem[j], segItem[j + 1])
  double* pc;
  double* tc;
  uint32_t* order;
  uint32_t* torder;
  const int4* item;   // (segment, begin, end, -)
  int* itemLower;     // per item: points <= split
  int* itemLowPre;    // per item: lower points of the segment's earlier items
  int* itemUpPre;     // per item: upper points of the segment's earlier items
  WideSeg* seg;
  double* outLo;
  double* outHi;
  double* outCenter;
  double* outRadius;
  int* outMid;
};

__device__ __forceinline__ unsigned long long wide_bmin(unsigned long long v, unsigned long long* scratch) {
  // block min of keys (the caller syncs around)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long r = scratch[0];
  for (int w = 1; w < kWideThreads / 32; ++w) r = min(r, scratch[w]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ unsigned long long wide_bmax(unsigned long long v, unsigned long long* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long r = scratch[0];
  for (int w = 1; w < kWideThreads / 32; ++w) r = max(r, scratch[w]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kWideThreads) wide_box(WideArgs A) {
  const int4 it = A.item[blockIdx.x];
  __shared__ unsigned long long sc[kWideThreads / 32];
  WideSeg& S = A.seg[it.x];
  for (int a = 0; a < A.d; ++a) {
    unsigned long long mn = ~0ull, mx = 0ull;
    const double* col = A.pc + static_cast<size_t>(a) * A.n;
    for (int pos = it.y + threadIdx.x; pos < it.z; pos += kWideThreads) {
      const unsigned long long k = toKey(col[pos]);
      mn = min(mn, k);
      mx = max(mx, k);
    }
    mn = wide_bmin(mn, sc);
    mx = wide_bmax(mx, sc);
    if (threadIdx.x == 0) {
      atomicMin(&S.boxKey[a][0], mn);
      atomicMax(&S.boxKey[a][1], mx);
    }
  }
}

// one thread per segment: tree.cpp:48-62 on the exact box
__global__ void wide_box_final(WideArgs A, int segOut0) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.ns) return;
  WideSeg& S = A.seg[s];
  const int d = A.d;
  double lo[FKTB_MAX_DIM], hi[FKTB_MAX_DIM];
  double extent = 0.0;
  for (int a = 0; a < d; ++a) {
    lo[a] = fromKey(S.boxKey[a][0]);
    hi[a] = fromKey(S.boxKey[a][1]);
    extent = extent + (hi[a] - lo[a]);
  }
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
  for (int a = 0; a < d; ++a) {
    S.ctr[a] = 0.5 * (lo[a] + hi[a]);
    const size_t o = static_cast<size_t>(A.outIdx[s]) * d + a;
    A.outLo[o] = lo[a];
    A.outHi[o] = hi[a];
    A.outCenter[o] = S.ctr[a];
  }
  S.extent = extent;
  S.r2Key = 0ull;
  (void)segOut0;
}

__global__ void __launch_bounds__(kWideThreads) wide_radius(WideArgs A) {
  const int4 it = A.item[blockIdx.x];
  __shared__ unsigned long long sc[kWideThreads / 32];
  WideSeg& S = A.seg[it.x];
  double ctr[FKTB_MAX_DIM];
  for (int a = 0; a < A.d; ++a) ctr[a] = S.ctr[a];
  double r2 = 0.0;
  for (int pos = it.y + threadIdx.x; pos < it.z; pos += kWideThreads) {
    double dist2 = 0.0;
    for (int a = 0; a < A.d; ++a) {
      const double t = A.pc[static_cast<size_t>(a) * A.n + pos] - ctr[a];
      dist2 = dist2 + t * t;
    }
    r2 = fmax(r2, dist2);
  }
  // r2 >= 0: its bit pattern orders like the value
  const unsigned long long m = wide_bmax(static_cast<unsigned long long>(__double_as_longlong(r2)), sc);
  if (threadIdx.x == 0) atomicMax(&S.r2Key, m);
}

// one thread per segment: radius, leaf test, axis and clamp (tree.cpp:64-115)
__global__ void wide_radius_final(WideArgs A) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.ns) return;
  WideSeg& S = A.seg[s];
  const int d = A.d;
  A.outRadius[A.outIdx[s]] = sqrt(__longlong_as_double(static_cast<long long>(S.r2Key)));
  const int cnt = S.end - S.begin;
  for (int i = 0; i < 256; ++i) S.hist[i] = 0;
  if (cnt <= A.leafCap || S.extent == 0.0) {
    S.active = 0;
    A.outMid[A.outIdx[s]] = -1;
    return;
  }
  S.active = 1;
  const double* lo = A.outLo + static_cast<size_t>(A.outIdx[s]) * d;
  const double* hi = A.outHi + static_cast<size_t>(A.outIdx[s]) * d;
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
  S.axis = axis;
  S.clampLo = cl;
  S.clampHi = ch;
  S.prefix = 0ull;
  S.k = cnt / 2;
}

__global__ void __launch_bounds__(kWideThreads) wide_hist(WideArgs A, int pass) {
  const int4 it = A.item[blockIdx.x];
  WideSeg& S = A.seg[it.x];
  if (!S.active) return;
  __shared__ unsigned hist[256];
  for (int i = threadIdx.x; i < 256; i += kWideThreads) hist[i] = 0;
  __syncthreads();
  const int shift = 56 - 8 * pass;
  const unsigned long long highMask = pass == 0 ? 0ull : (~0ull << (shift + 8));
  const unsigned long long prefix = S.prefix;
  const double* col = A.pc + static_cast<size_t>(S.axis) * A.n;
  for (int pos = it.y + threadIdx.x; pos < it.z; pos += kWideThreads) {
    const unsigned long long key = toKey(col[pos]);
    if ((key & highMask) == prefix) atomicAdd(&hist[(key >> shift) & 255ull], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += kWideThreads)
    if (hist[i]) atomicAdd(&S.hist[i], hist[i]);
}

// one thread per segment: the digit holding the k-th smallest key
__global__ void wide_select(WideArgs A, int pass) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.ns) return;
  WideSeg& S = A.seg[s];
  if (!S.active) return;
  const int shift = 56 - 8 * pass;
  unsigned cum = 0;
  const int k = S.k;
  for (int dg = 0; dg < 256; ++dg) {
    if (cum + S.hist[dg] > static_cast<unsigned>(k)) {
      S.prefix |= static_cast<unsigned long long>(dg) << shift;
      S.k = k - static_cast<int>(cum);
      break;
    }
    cum += S.hist[dg];
  }
  for (int i = 0; i < 256; ++i) S.hist[i] = 0;
  if (pass == 7) {
    const double v = fromKey(S.prefix);
    S.split = v < S.clampLo ? S.clampLo : (S.clampHi < v ? S.clampHi : v);  // std::clamp
    S.lower = 0ull;
    S.mxKey = 0ull;
    S.belowKey = 0ull;
  }
}

// MODE 0: lower counts; 1: max (fallback); 2: largest value below the max;
// 3: lower counts again at the fallback split
template <int MODE>
__global__ void __launch_bounds__(kWideThreads) wide_scan(WideArgs A) {
  const int4 it = A.item[blockIdx.x];
  WideSeg& S = A.seg[it.x];
  if (!S.active || (MODE > 0 && !S.fallback)) return;
  __shared__ long long sl[32];
  __shared__ unsigned long long sc[kWideThreads / 32];
  const double* col = A.pc + static_cast<size_t>(S.axis) * A.n;
  if constexpr (MODE == 0 || MODE == 3) {
    const double split = S.split;
    long long lower = 0;
    for (int pos = it.y + threadIdx.x; pos < it.z; pos += kWideThreads) lower += col[pos] <= split ? 1 : 0;
    lower = block_sum_ll(lower, sl);
    if (threadIdx.x == 0) {
      A.itemLower[blockIdx.x] = static_cast<int>(lower);
      atomicAdd(&S.lower, static_cast<unsigned long long>(lower));
    }
  } else {
    const double mx = MODE == 2 ? fromKey(S.mxKey) : 0.0;
    unsigned long long m = 0ull;
    for (int pos = it.y + threadIdx.x; pos < it.z; pos += kWideThreads) {
      const double v = col[pos];
      if (MODE == 1 || v < mx) m = max(m, toKey(v));
    }
    m = wide_bmax(m, sc);
    if (threadIdx.x == 0) atomicMax(MODE == 1 ? &S.mxKey : &S.belowKey, m);
  }
}

// one thread per segment: all points on one side -> fallback split
// (tree.cpp:136-159); after the recount, per-item prefixes and the midpoint
__global__ void wide_check(WideArgs A, int stage) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.ns) return;
  WideSeg& S = A.seg[s];
  if (!S.active) return;
  const unsigned long long cnt = static_cast<unsigned long long>(S.end - S.begin);
  if (stage == 0) {
    S.fallback = S.lower == 0 || S.lower == cnt;
  } else if (stage == 1) {
    if (S.fallback) {
      S.split = fromKey(S.belowKey);
      S.lower = 0ull;
    }
  }
}

__global__ void wide_prefix(WideArgs A) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.ns) return;
  WideSeg& S = A.seg[s];
  if (!S.active) return;
  int low = 0, up = 0;
  for (int i = A.segItem[s]; i < A.segItem[s + 1]; ++i) {
    const int4 it = A.item[i];
    A.itemLowPre[i] = low;
    A.itemUpPre[i] = up;
    low += A.itemLower[i];
    up += (it.z - it.y) - A.itemLower[i];
  }
  A.outMid[A.outIdx[s]] = S.begin + low;
}

// stable partition of one item's range (ballot / popc scan per chunk)
__global__ void __launch_bounds__(kWideThreads) wide_partition(WideArgs A) {
  const int4 it = A.item[blockIdx.x];
  WideSeg& S = A.seg[it.x];
  if (!S.active) return;
  __shared__ int warpCnt[kWideThreads / 32];
  const int n = A.n, d = A.d;
  const double split = S.split;
  const double* col = A.pc + static_cast<size_t>(S.axis) * n;
  const int L = static_cast<int>(S.lower);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kWideThreads / 32;
  int lowerBase = S.begin + A.itemLowPre[blockIdx.x];
  int upperBase = S.begin + L + A.itemUpPre[blockIdx.x];
  for (int start = it.y; start < it.z; start += kWideThreads) {
    const int pos = start + threadIdx.x;
    const bool valid = pos < it.z;
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
      const int dst = flag ? lowerBase + before : upperBase + (pos - start - before);
      for (int a = 0; a < d; ++a) A.tc[static_cast<size_t>(a) * n + dst] = A.pc[static_cast<size_t>(a) * n + pos];
      A.torder[dst] = A.order[pos];
    }
    const int chunk = min(kWideThreads, it.z - start);
    lowerBase += chunkLower;
    upperBase += chunk - chunkLower;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kWideThreads) wide_copyback(WideArgs A) {
  const int4 it = A.item[blockIdx.x];
  if (!A.seg[it.x].active) return;
  for (int pos = it.y + threadIdx.x; pos < it.z; pos += kWideThreads) {
    for (int a = 0; a < A.d; ++a) A.pc[static_cast<size_t>(a) * A.n + pos] = A.tc[static_cast<size_t>(a) * A.n + pos];
    A.order[pos] = A.torder[pos];
  }
}

__global__ void wide_init(WideArgs A, const int* segB, const int* segE) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= A.ns) return;
  WideSeg& S = A.seg[s];
  for (int a = 0; a < A.d; ++a) {
    S.boxKey[a][0] = ~0ull;
    S.boxKey[a][1] = 0ull;
  }
  S.begin = segB[s];
  S.end = segE[s];
  S.active = 0;
  S.fallback = 0;
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
                    DeviceBuffer<uint32_t>& keysOut, DeviceBuffer<unsigned char>& temp, cudaStream_t st) {
  dOff.resize(static_cast<size_t>(nodes) + 1);
  outPos.resize(static_cast<size_t>(std::max<long long>(total, 1)));
  hOff.assign(static_cast<size_t>(nodes) + 1, 0);
  if (total == 0) {
    FKTB_CUDA(cudaMemsetAsync(dOff.get(), 0, dOff.bytes(), st));
    return;
  }
  keysOut.resize(static_cast<size_t>(total));
  size_t tempBytes = 0;
  FKTB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tempBytes, keys.get(), keysOut.get(), vals.get(), outPos.get(),
                                            static_cast<int64_t>(total), 0, bitsFor(nodes), st));
  temp.resize(tempBytes);
  FKTB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tempBytes, keys.get(), keysOut.get(), vals.get(),
                                            outPos.get(), static_cast<int64_t>(total), 0, bitsFor(nodes), st));
  csr_offsets<<<(nodes + 1 + 255) / 256, 256, 0, st>>>(keysOut.get(), total, nodes, dOff.get());
  FKTB_CUDA(cudaGetLastError());
  FKTB_CUDA(cudaMemcpyAsync(hOff.data(), dOff.get(), dOff.bytes(), cudaMemcpyDeviceToHost, st));
  FKTB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void buildTreeGpu(DeviceTree& t, const double* hostX, int n, int d, int leafCapacity, cudaStream_t st,
                  const double* devX) {
  if (leafCapacity < 1) throw std::invalid_argument("leaf capacity must be >= 1");
  if (n < 1) throw std::invalid_argument("point cloud must be nonempty");
  if (d < 1 || d > FKTB_MAX_DIM) throw std::invalid_argument("GPU tree supports 1 <= d <= 16");
  t.n = n;
  t.d = d;
  t.leafCapacity = leafCapacity;
  t.stream = st;
  const size_t nd = static_cast<size_t>(n) * d;
  auto& S = t.scratch;
  DeviceBuffer<double>& x = S.x;
  DeviceBuffer<double>& tc = S.tc;
  DeviceBuffer<uint32_t>& torder = S.torder;
  x.resize(devX ? 0 : nd);
  tc.resize(nd);
  torder.resize(static_cast<size_t>(n));
  t.pc.resize(nd);
  t.order.resize(static_cast<size_t>(n));
  if (!devX) FKTB_CUDA(cudaMemcpyAsync(x.get(), hostX, nd * sizeof(double), cudaMemcpyHostToDevice, st));
  transpose_to_soa<<<(n + 255) / 256, 256, 0, st>>>(devX ? devX : x.get(), n, d, t.pc.get(), t.order.get());
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
  DeviceBuffer<int>& dSegB = S.segB;
  DeviceBuffer<int>& dSegE = S.segE;
  DeviceBuffer<int>& dMid = S.mid;
  dSegB.resize(static_cast<size_t>(maxSeg));
  dSegE.resize(static_cast<size_t>(maxSeg));
  dMid.resize(static_cast<size_t>(maxSeg));
  DeviceBuffer<double>& dLo = S.lo;
  DeviceBuffer<double>& dHi = S.hi;
  DeviceBuffer<double>& dC = S.c;
  DeviceBuffer<double>& dR = S.r;
  dLo.resize(static_cast<size_t>(maxSeg) * d);
  dHi.resize(static_cast<size_t>(maxSeg) * d);
  dC.resize(static_cast<size_t>(maxSeg) * d);
  dR.resize(static_cast<size_t>(maxSeg));
  std::vector<int> hb, he, hmid;
  std::vector<int4> hItems;
  std::vector<int> hWideB, hWideE, hWideOut, hNarB, hNarE, hNarOut, hSegItem;
  DeviceBuffer<int4>& dItems = S.items;
  DeviceBuffer<int>& dItemLower = S.itemLower;
  DeviceBuffer<int>& dItemLowPre = S.itemLowPre;
  DeviceBuffer<int>& dItemUpPre = S.itemUpPre;
  const size_t maxWide = static_cast<size_t>(n / kWideMin + 2);
  S.wide.resize(maxWide * sizeof(WideSeg));
  WideSeg* dWide = reinterpret_cast<WideSeg*>(S.wide.get());
  DeviceBuffer<int>& dWideB = S.wideB;
  DeviceBuffer<int>& dWideE = S.wideE;
  DeviceBuffer<int>& dWideOut = S.wideOut;
  DeviceBuffer<int>& dSegItem = S.segItem;
  DeviceBuffer<int>& dNarOut = S.narOut;
  dWideB.resize(maxWide);
  dWideE.resize(maxWide);
  dWideOut.resize(maxWide);
  dSegItem.resize(maxWide + 1);
  dNarOut.resize(static_cast<size_t>(maxSeg));
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
    // segments above kWideMin points take the wide (multi-CTA) path, the
    // rest one CTA each; both write the level slots of their segments
    hWideB.clear();
    hWideE.clear();
    hWideOut.clear();
    hNarB.clear();
    hNarE.clear();
    hNarOut.clear();
    for (int i = 0; i < ns; ++i) {
      const bool wide = he[i] - hb[i] > kWideMin;
      (wide ? hWideB : hNarB).push_back(hb[i]);
      (wide ? hWideE : hNarE).push_back(he[i]);
      (wide ? hWideOut : hNarOut).push_back(i);
    }
    if (!hNarB.empty()) {
      const int nn = static_cast<int>(hNarB.size());
      FKTB_CUDA(cudaMemcpyAsync(dSegB.get(), hNarB.data(), nn * sizeof(int), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dSegE.get(), hNarE.data(), nn * sizeof(int), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dNarOut.get(), hNarOut.data(), nn * sizeof(int), cudaMemcpyHostToDevice, st));
      LevelArgs A{n,        d,           leafCapacity, t.pc.get(), tc.get(), t.order.get(), torder.get(), dSegB.get(),
                  dSegE.get(), dNarOut.get(), dLo.get(),    dHi.get(),  dC.get(),  dR.get(),      dMid.get()};
      tree_level_kernel<<<nn, kTreeThreads, 0, st>>>(A);
      FKTB_CUDA(cudaGetLastError());
    }
    if (!hWideB.empty()) {
      const int nw = static_cast<int>(hWideB.size());
      hItems.clear();
      hSegItem.assign(1, 0);
      for (int i = 0; i < nw; ++i) {
        for (int b0 = hWideB[i];; b0 += kWideItem) {
          hItems.push_back(make_int4(i, b0, std::min(hWideE[i], b0 + kWideItem), 0));
          if (b0 + kWideItem >= hWideE[i]) break;
        }
        hSegItem.push_back(static_cast<int>(hItems.size()));
      }
      const int items = static_cast<int>(hItems.size());
      if (dItems.size() < hItems.size()) {
        dItems.resize(hItems.size());
        dItemLower.resize(hItems.size());
        dItemLowPre.resize(hItems.size());
        dItemUpPre.resize(hItems.size());
      }
      FKTB_CUDA(cudaMemcpyAsync(dItems.get(), hItems.data(), hItems.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dWideB.get(), hWideB.data(), nw * sizeof(int), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dWideE.get(), hWideE.data(), nw * sizeof(int), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dWideOut.get(), hWideOut.data(), nw * sizeof(int), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dSegItem.get(), hSegItem.data(), hSegItem.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      WideArgs W{n, d, leafCapacity, nw, items, dWideOut.get(), dSegItem.get(), t.pc.get(), tc.get(), t.order.get(),
                 torder.get(), dItems.get(), dItemLower.get(), dItemLowPre.get(), dItemUpPre.get(), dWide,
                 dLo.get(), dHi.get(), dC.get(), dR.get(), dMid.get()};
      const int sb = (nw + 127) / 128;
      wide_init<<<sb, 128, 0, st>>>(W, dWideB.get(), dWideE.get());
      wide_box<<<items, kWideThreads, 0, st>>>(W);
      wide_box_final<<<sb, 128, 0, st>>>(W, 0);
      wide_radius<<<items, kWideThreads, 0, st>>>(W);
      wide_radius_final<<<sb, 128, 0, st>>>(W);
      for (int pass = 0; pass < 8; ++pass) {
        wide_hist<<<items, kWideThreads, 0, st>>>(W, pass);
        wide_select<<<sb, 128, 0, st>>>(W, pass);
      }
      wide_scan<0><<<items, kWideThreads, 0, st>>>(W);
      wide_check<<<sb, 128, 0, st>>>(W, 0);
      wide_scan<1><<<items, kWideThreads, 0, st>>>(W);
      wide_scan<2><<<items, kWideThreads, 0, st>>>(W);
      wide_check<<<sb, 128, 0, st>>>(W, 1);
      wide_scan<3><<<items, kWideThreads, 0, st>>>(W);
      wide_prefix<<<sb, 128, 0, st>>>(W);
      wide_partition<<<items, kWideThreads, 0, st>>>(W);
      wide_copyback<<<items, kWideThreads, 0, st>>>(W);
    }
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

  auto& S = t.scratch;
  DeviceBuffer<int>& farCnt = S.farCnt;
  DeviceBuffer<int>& nearCnt = S.nearCnt;
  DeviceBuffer<long long>& farStart = S.farStart;
  DeviceBuffer<long long>& nearStart = S.nearStart;
  farCnt.resize(static_cast<size_t>(n));
  nearCnt.resize(static_cast<size_t>(n));
  farStart.resize(static_cast<size_t>(n) + 1);
  nearStart.resize(static_cast<size_t>(n) + 1);
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
    DeviceBuffer<unsigned char>& temp = S.temp;
    temp.resize(bytes);
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, farCnt.get(), farStart.get() + 1, n, st));
    FKTB_CUDA(cub::DeviceScan::InclusiveSum(temp.get(), bytes, nearCnt.get(), nearStart.get() + 1, n, st));
  }
  long long totals[2] = {0, 0};
  FKTB_CUDA(cudaMemcpyAsync(&totals[0], farStart.get() + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FKTB_CUDA(cudaMemcpyAsync(&totals[1], nearStart.get() + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FKTB_CUDA(cudaStreamSynchronize(st));
  t.farTotal = totals[0];
  t.nearTotal = totals[1];
  DeviceBuffer<uint32_t>& farNode = S.farNode;
  DeviceBuffer<uint32_t>& farPos = S.farPos;
  DeviceBuffer<uint32_t>& nearNode = S.nearNode;
  DeviceBuffer<uint32_t>& nearPos = S.nearPos;
  farNode.resize(static_cast<size_t>(std::max(1ll, t.farTotal)));
  farPos.resize(static_cast<size_t>(std::max(1ll, t.farTotal)));
  nearNode.resize(static_cast<size_t>(std::max(1ll, t.nearTotal)));
  nearPos.resize(static_cast<size_t>(std::max(1ll, t.nearTotal)));
  A.farStart = farStart.get();
  A.nearStart = nearStart.get();
  A.farNode = farNode.get();
  A.farPos = farPos.get();
  A.nearNode = nearNode.get();
  A.nearPos = nearPos.get();
  sets_kernel<1><<<blocks, 128, 0, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
  sortPairsToCsr(farNode, farPos, t.farTotal, nodes, t.dFarOff, t.farOff, t.dFarPos, S.keysOut, S.temp, st);
  sortPairsToCsr(nearNode, nearPos, t.nearTotal, nodes, t.dNearOff, t.nearOff, t.dNearPos, S.keysOut, S.temp, st);
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
