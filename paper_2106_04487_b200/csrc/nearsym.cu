// K3 near field, symmetric blocks (FP64).
//
// The reference evaluates z_t += sum_{s in l} K(|x_t - x_s|) y_s for every
// leaf l and t in N_l (transform.cpp:163-181). For two leaves A != B let
// T_AB = N_A ∩ B (targets in B that need A's sources). Every pair
// (t in T_AB, s in T_BA) is near in both directions, so K(t, s) is evaluated
// once and feeds both z_t += K y_s and z_s += K y_t (the value is the same:
// (x_t - x_s)^2 == (x_s - x_t)^2 bitwise). The rest of each leaf pair is
// one-way: rows T_AB against A \ T_BA, rows T_BA against B \ T_AB, rows
// N_A ∩ A against A. At cfg2 ~2/3 of all near pairs are mutual, so kernel
// evaluations drop by ~1/3 with the same sums (up to the order of the FP64
// atomic accumulation).
//
// Blocks are lists of permuted positions in one index pool:
//   [ near-set positions (the CSR of K2) | identity 0..n-1 | extra lists ]
// The extra lists are the complements A \ T_BA and, per leaf, the merged rows
// that need all of the leaf's sources (non-mutual targets and the leaf's own),
// so those form one long row list instead of many short ones.
// Tiles: <= 256 rows x all columns. Warp w owns rows [128w, 128w + 128) in
// groups of 32 (warp-uniform group count), so short row sets pad to 32, not
// 256. Columns are staged in shared memory (512 at a time one-way, 32 in
// symmetric tiles); in symmetric tiles every thread stores its per-column
// partial to shared memory and the column sums go to z with one atomic per
// column per tile.
#include <algorithm>
#include <cstdlib>
#include <unordered_map>

#include "fastmath.cuh"
#include "near_common.cuh"
#include "plan.hpp"

namespace fktb {
namespace {

constexpr int kSymThreads = 64;
constexpr int kSymTPT = 4;
constexpr int kSymRows = kSymThreads * kSymTPT;
constexpr int kSymChunk = 512;    // columns staged per pass, one-way tiles
constexpr int kSymChunkS = 32;    // columns per pass in symmetric tiles
constexpr int kZsStride = kSymThreads + 1;

struct SymArgs {
  int n;
  const double* pc;
  const uint32_t* pool;
  const FktbBlockTile* tiles;
  const double* yp;
  double* zp;
  const double* expTable;
  double sc, wf, diagCanon;
};

template <int KID, int D, bool SEL, bool SYM>
__device__ __forceinline__ void block_body(const SymArgs& A, const FktbBlockTile& tile, double* ss, double* zs,
                                           const double* tab) {
  constexpr int SP = (D + 2) / 2 * 2;
  const int n = A.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wRows = min(max(tile.rowCount - warp * 32 * kSymTPT, 0), 32 * kSymTPT);
  const int groups = (wRows + 31) >> 5;  // warp-uniform
  const int activeThreads = tile.rowCount > 32 * kSymTPT ? kSymThreads : 32;
  int tpos[kSymTPT];
  double tx[kSymTPT][D];
  double ty[kSymTPT];
  double acc[kSymTPT];
#pragma unroll
  for (int i = 0; i < kSymTPT; ++i) {
    const int idx = warp * 32 * kSymTPT + i * 32 + lane;
    tpos[i] = idx < tile.rowCount ? static_cast<int>(A.pool[tile.rowOff + idx]) : -1;
    const int p = tpos[i] >= 0 ? tpos[i] : 0;
#pragma unroll
    for (int a = 0; a < D; ++a) tx[i][a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + p], A.sc);  // uncontracted (see near.cu)
    ty[i] = tpos[i] >= 0 ? A.yp[p] * A.wf : 0.0;
    acc[i] = 0.0;
  }
  constexpr int CH = SYM ? kSymChunkS : kSymChunk;
  for (int cs = 0; cs < tile.colCount; cs += CH) {
    const int cn = min(CH, tile.colCount - cs);
    __syncthreads();
    for (int s = threadIdx.x; s < cn; s += kSymThreads) {
      const int pos = static_cast<int>(A.pool[tile.colOff + cs + s]);
#pragma unroll
      for (int a = 0; a < D; ++a) ss[s * SP + a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + pos], A.sc);
      ss[s * SP + D] = A.yp[pos] * A.wf;
    }
    __syncthreads();
#pragma unroll 2
    for (int s = 0; s < (groups > 0 ? cn : 0); ++s) {
      double src[SP];
#pragma unroll
      for (int q = 0; q < SP; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(&ss[s * SP + q]);
        src[q] = v.x;
        src[q + 1] = v.y;
      }
      double part = 0.0;
#pragma unroll
      for (int i = 0; i < kSymTPT; ++i) {
        if (i >= groups) break;
        const double d0 = tx[i][0] - src[0];
        double q = fma(d0, d0, kQBias);
#pragma unroll
        for (int a = 1; a < D; ++a) {
          const double da = tx[i][a] - src[a];
          q = fma(da, da, q);
        }
        double kv = FastKernel<KID>::template eval<1>(q, tab);
        if constexpr (SEL) kv = q == kQBias ? A.diagCanon : kv;
        acc[i] = fma(kv, src[D], acc[i]);
        if constexpr (SYM) part = fma(kv, ty[i], part);
      }
      if constexpr (SYM) zs[s * kZsStride + threadIdx.x] = part;  // per-thread partial, reduced below
    }
    if constexpr (SYM) {
      __syncthreads();
      for (int s = threadIdx.x; s < cn; s += kSymThreads) {
        double t = 0.0;
#pragma unroll 8
        for (int j = 0; j < activeThreads; ++j) t += zs[s * kZsStride + j];
        atomicAdd(A.zp + A.pool[tile.colOff + cs + s], t);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kSymTPT; ++i)
    if (tpos[i] >= 0) atomicAdd(A.zp + tpos[i], acc[i]);
}

template <int KID, int D, bool SEL>
__global__ void __launch_bounds__(kSymThreads, 10) near_block_kernel(const __grid_constant__ SymArgs A) {
  constexpr int SP = (D + 2) / 2 * 2;
  // one-way tiles: ss[512 * SP]; symmetric tiles: ss[32 * SP] then zs[32 x 65]
  constexpr int kOne = kSymChunk * SP, kSym = kSymChunkS * (SP + kZsStride);
  __shared__ __align__(16) double ss[kOne > kSym ? kOne : kSym];
  double* zs = ss + kSymChunkS * SP;
  __shared__ double tab[kNearExpTable];
  if constexpr (FastKernel<KID>::needsTable)
    for (int i = threadIdx.x; i < kNearExpTable; i += kSymThreads) tab[i] = A.expTable[i];
  const FktbBlockTile tile = A.tiles[blockIdx.x];
  if (tile.sym)
    block_body<KID, D, SEL, true>(A, tile, ss, zs, tab);
  else
    block_body<KID, D, SEL, false>(A, tile, ss, zs, tab);
}

template <int KID, int D>
void launchSymT(const SymArgs& A, bool sel, int tiles, cudaStream_t st) {
  if (sel)
    near_block_kernel<KID, D, true><<<tiles, kSymThreads, 0, st>>>(A);
  else
    near_block_kernel<KID, D, false><<<tiles, kSymThreads, 0, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

template <int KID>
bool launchSymK(const SymArgs& A, int d, bool sel, int tiles, cudaStream_t st) {
  if constexpr (!FastKernel<KID>::supported) {
    return false;
  } else {
    switch (d) {
      case 2: launchSymT<KID, 2>(A, sel, tiles, st); return true;
      case 3: launchSymT<KID, 3>(A, sel, tiles, st); return true;
      case 5: launchSymT<KID, 5>(A, sel, tiles, st); return true;
      default: return false;
    }
  }
}

// ---------------------------------------------------------------------------
// Symmetric blocks in the Gram form (near.cu near_tile): one
// warp per tile, lane owning rows lane + 32 i (i < G, G = ceil(rows / 32)
// chosen per tile by a switch so every instantiation keeps G independent
// chains); columns staged in shared memory 128 at a time as (-2 s, |s|^2 +
// offset + bias, weight). In symmetric tiles each lane also accumulates
// K(t_i, s) y_t over its rows; a 5-step butterfly gives the column sum, and
// the chunk's column sums go to z with one atomic per column.
struct SymGArgs {
  int n;
  const double* pc;
  const uint32_t* pool;
  const FktbBlockTile* tiles;
  const double* yp;
  double* zp;
  const double* expTable;
  double sc, wf;
  const double* center;
  const double* limit2;
  double gramLimit2;  // tile bound B = limit2[leaf] * kGramBoundSym / gramLimit2
};

constexpr double kGramBoundSym = 128.0;  // as near.cu kGramBound
constexpr int kSymGChunk = 128;

template <int KID, int D, bool SYM, int G>
__device__ __forceinline__ void gram_block(const SymGArgs& A, const FktbBlockTile& tile, double* ss, double* colbuf,
                                           int* colpos, const double* tab) {
  using FK = FastKernel<KID>;
  constexpr int SP = (D + 2 + 1) / 2 * 2;
  const int n = A.n;
  const int lane = threadIdx.x & 31;
  const int leaf = tile.leaf;
  double c[D];
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = A.center[static_cast<size_t>(leaf) * D + a];
  const double wfG = A.wf * FK::gramWeight;
  const double qbias = FK::gramBiased
                           ? fma((1.5 * D + 1.0) * 2.220446049250313e-16 * kGramBoundSym / A.gramLimit2, A.limit2[leaf], 1e-30)
                           : 0.0;
  int tpos[G];
  double tx[G][D], tn[G], ty[G], acc[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int idx = i * 32 + lane;
    tpos[i] = idx < tile.rowCount ? static_cast<int>(A.pool[tile.rowOff + idx]) : -1;
    const int p = tpos[i] >= 0 ? tpos[i] : static_cast<int>(A.pool[tile.rowOff]);  // dead lanes: a copy of row 0
    tn[i] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      tx[i][a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + p] - c[a], A.sc);
      tn[i] = fma(tx[i][a], tx[i][a], tn[i]);
    }
    ty[i] = SYM && tpos[i] >= 0 ? A.yp[p] * wfG : 0.0;
    acc[i] = 0.0;
  }
  for (int cs = 0; cs < tile.colCount; cs += kSymGChunk) {
    const int cn = min(kSymGChunk, tile.colCount - cs);
    __syncwarp();
    for (int s = lane; s < cn; s += 32) {
      const int pos = static_cast<int>(A.pool[tile.colOff + cs + s]);
      double ns = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double v = __dmul_rn(A.pc[static_cast<size_t>(a) * n + pos] - c[a], A.sc);
        ns = fma(v, v, ns);
        ss[s * SP + a] = -2.0 * v;
      }
      ss[s * SP + D] = ns + (FK::gramOffset + qbias);
      ss[s * SP + D + 1] = A.yp[pos] * wfG;
      if constexpr (SYM) colpos[s] = pos;
    }
    __syncwarp();
#pragma unroll 2
    for (int s = 0; s < cn; ++s) {
      double src[SP];
#pragma unroll
      for (int q = 0; q < SP; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(&ss[s * SP + q]);
        src[q] = v.x;
        src[q + 1] = v.y;
      }
      double cp = 0.0;
#pragma unroll
      for (int i = 0; i < G; ++i) {
        double q = fma(tx[i][0], src[0], src[D]);
#pragma unroll
        for (int a = 1; a < D; ++a) q = fma(tx[i][a], src[a], q);
        q += tn[i];
        const double kv = FK::template eval<kNearExpRep, true, true>(q, tab, 0);
        acc[i] = fma(kv, src[D + 1], acc[i]);
        if constexpr (SYM) cp = fma(kv, ty[i], cp);
      }
      if constexpr (SYM) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cp += __shfl_xor_sync(0xffffffffu, cp, o);
        if (lane == (s & 31)) colbuf[s] = cp;
      }
    }
    if constexpr (SYM) {
      __syncwarp();
      for (int s = lane; s < cn; s += 32) atomicAdd(A.zp + colpos[s], colbuf[s]);
    }
  }
#pragma unroll
  for (int i = 0; i < G; ++i)
    if (tpos[i] >= 0) atomicAdd(A.zp + tpos[i], acc[i]);
}

template <int KID, int D, bool SYM>
__device__ __forceinline__ void gram_block_g(const SymGArgs& A, const FktbBlockTile& tile, double* ss, double* colbuf,
                                             int* colpos, const double* tab) {
  switch ((tile.rowCount + 31) >> 5) {  // warp-uniform
    case 1: return gram_block<KID, D, SYM, 1>(A, tile, ss, colbuf, colpos, tab);
    case 2: return gram_block<KID, D, SYM, 2>(A, tile, ss, colbuf, colpos, tab);
    case 3: return gram_block<KID, D, SYM, 3>(A, tile, ss, colbuf, colpos, tab);
    case 4: return gram_block<KID, D, SYM, 4>(A, tile, ss, colbuf, colpos, tab);
    case 5: return gram_block<KID, D, SYM, 5>(A, tile, ss, colbuf, colpos, tab);
    case 6: return gram_block<KID, D, SYM, 6>(A, tile, ss, colbuf, colpos, tab);
    case 7: return gram_block<KID, D, SYM, 7>(A, tile, ss, colbuf, colpos, tab);
    default: return gram_block<KID, D, SYM, 8>(A, tile, ss, colbuf, colpos, tab);
  }
}

template <int KID, int D>
__global__ void __launch_bounds__(32) near_sym_gram(const __grid_constant__ SymGArgs A) {
  static_assert(kSymRows == 256, "block tiles of 256 rows = 32 lanes x 8");
  constexpr int SP = (D + 2 + 1) / 2 * 2;
  __shared__ __align__(16) double ss[kSymGChunk * SP];
  __shared__ double colbuf[kSymGChunk];
  __shared__ int colpos[kSymGChunk];
  __shared__ double tab[kNearExpTable * kNearExpRep];
  if constexpr (FastKernel<KID>::needsTable)
    for (int i = threadIdx.x; i < kNearExpTable * kNearExpRep; i += 32) tab[i] = A.expTable[i / kNearExpRep];
  __syncwarp();
  const FktbBlockTile tile = A.tiles[blockIdx.x];
  if (tile.sym)
    gram_block_g<KID, D, true>(A, tile, ss, colbuf, colpos, tab);
  else
    gram_block_g<KID, D, false>(A, tile, ss, colbuf, colpos, tab);
}

bool symSupported(int kid, int d) {
  const bool k = kid == FKTB_KERNEL_MATERN32 || kid == FKTB_KERNEL_MATERN12 || kid == FKTB_KERNEL_EXPONENTIAL ||
                 kid == FKTB_KERNEL_CAUCHY || kid == FKTB_KERNEL_RATIONAL_QUADRATIC || kid == FKTB_KERNEL_GAUSSIAN ||
                 kid == FKTB_KERNEL_INVERSE_R || kid == FKTB_KERNEL_INVERSE_R2;
  return k && (d == 2 || d == 3 || d == 5);
}

}  // namespace

void buildNearBlocks(DevicePlan& plan, bool oneWayOnly) {
  const DeviceTree& t = *plan.tree;
  if (!symSupported(plan.kernel.id, plan.d) || t.nearTotal == 0) return;
  const int n = t.n;
  // host copy of the near CSR (positions ascending per leaf)
  std::vector<uint32_t> nearPos(static_cast<size_t>(t.nearTotal));
  FKTB_CUDA(cudaMemcpy(nearPos.data(), t.dNearPos.get(), nearPos.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  std::vector<int> leafOf(static_cast<size_t>(n), -1);
  for (int b = 0; b < t.nodes; ++b)
    if (t.left[static_cast<size_t>(b)] < 0)
      for (uint32_t p = t.begin[static_cast<size_t>(b)]; p < t.end[static_cast<size_t>(b)]; ++p) leafOf[p] = b;
  // segments: leaf A's near list grouped by the leaf of the target
  struct Seg {
    long long off;
    int len;
  };
  std::unordered_map<unsigned long long, Seg> seg;
  std::vector<std::vector<std::pair<int, Seg>>> segsOf(static_cast<size_t>(t.nodes));
  auto key = [](int a, int b) { return (static_cast<unsigned long long>(a) << 32) | static_cast<unsigned>(b); };
  for (int A = 0; A < t.nodes; ++A) {
    const long long o0 = t.nearOff[static_cast<size_t>(A)], o1 = t.nearOff[static_cast<size_t>(A) + 1];
    long long i = o0;
    while (i < o1) {
      const int B = leafOf[nearPos[static_cast<size_t>(i)]];
      long long j = i;
      while (j < o1 && leafOf[nearPos[static_cast<size_t>(j)]] == B) ++j;
      const Seg s{i, static_cast<int>(j - i)};
      seg[key(A, B)] = s;
      segsOf[static_cast<size_t>(A)].push_back({B, s});
      i = j;
    }
  }
  const long long identityBase = t.nearTotal;
  std::vector<uint32_t> comp;  // complements, appended after identity
  std::vector<FktbBlockTile> tiles;
  long long symPairs = 0, oneWay = 0;
  auto addBlock = [&](long long rowOff, int rowCount, long long colOff, int colCount, int sym, int leaf) {
    if (rowCount <= 0 || colCount <= 0) return;
    for (int r = 0; r < rowCount; r += kSymRows)
      tiles.push_back(FktbBlockTile{rowOff + r, colOff, std::min(kSymRows, rowCount - r), colCount, sym, leaf});
    (sym ? symPairs : oneWay) += static_cast<long long>(rowCount) * colCount;
  };
  auto complement = [&](int leaf, const Seg& sub) {
    // positions of leaf not in nearPos[sub], ascending; returns pool offset
    const long long base = identityBase + n + static_cast<long long>(comp.size());
    long long k = sub.off, kend = sub.off + sub.len;
    for (uint32_t p = t.begin[static_cast<size_t>(leaf)]; p < t.end[static_cast<size_t>(leaf)]; ++p) {
      if (k < kend && nearPos[static_cast<size_t>(k)] == p) {
        ++k;
        continue;
      }
      comp.push_back(p);
    }
    return std::make_pair(base, static_cast<int>(identityBase + n + static_cast<long long>(comp.size()) - base));
  };
  for (int A = 0; A < t.nodes; ++A) {
    if (t.left[static_cast<size_t>(A)] >= 0) continue;
    const long long aBegin = t.begin[static_cast<size_t>(A)];
    const int aCount = static_cast<int>(t.end[static_cast<size_t>(A)] - t.begin[static_cast<size_t>(A)]);
    if (oneWayOnly) {  // A/B: the same kernel on the plain leaf decomposition
      addBlock(t.nearOff[static_cast<size_t>(A)], static_cast<int>(t.nearOff[static_cast<size_t>(A) + 1] - t.nearOff[static_cast<size_t>(A)]),
               identityBase + aBegin, aCount, 0, A);
      continue;
    }
    // rows that need all of A's sources: A's own and non-mutual targets, merged
    const long long fullBase = identityBase + n + static_cast<long long>(comp.size());
    for (const auto& [B, sAB] : segsOf[static_cast<size_t>(A)])
      if (B == A || seg.find(key(B, A)) == seg.end())
        comp.insert(comp.end(), nearPos.begin() + sAB.off, nearPos.begin() + sAB.off + sAB.len);
    addBlock(fullBase, static_cast<int>(identityBase + n + static_cast<long long>(comp.size()) - fullBase),
             identityBase + aBegin, aCount, 0, A);
    for (const auto& [B, sAB] : segsOf[static_cast<size_t>(A)]) {
      if (B == A) continue;
      auto it = seg.find(key(B, A));
      if (it == seg.end()) continue;
      if (A > B) continue;  // mutual pair handled once, from the smaller leaf id
      const Seg& sBA = it->second;  // rows in A that need B's sources
      const long long bBegin = t.begin[static_cast<size_t>(B)];
      (void)bBegin;
      // rows T_AB (in B, near A) x cols T_BA (in A): centred on A, whose
      // bound covers both (rows within radius_A / theta, cols within radius_A)
      addBlock(sAB.off, sAB.len, sBA.off, sBA.len, 1, A);
      const auto cA = complement(A, sBA);              // A \ T_BA
      addBlock(sAB.off, sAB.len, cA.first, cA.second, 0, A);
      const auto cB = complement(B, sAB);              // B \ T_AB
      addBlock(sBA.off, sBA.len, cB.first, cB.second, 0, B);
    }
  }
  // Longest tiles first: the heavy symmetric blocks start early.
  std::stable_sort(tiles.begin(), tiles.end(), [](const FktbBlockTile& a, const FktbBlockTile& b) {
    return static_cast<long long>(a.rowCount) * a.colCount * (a.sym ? 2 : 1) >
           static_cast<long long>(b.rowCount) * b.colCount * (b.sym ? 2 : 1);
  });
  // pool = near positions | identity | complements
  const size_t poolSize = static_cast<size_t>(t.nearTotal) + n + comp.size();
  plan.dNearPool.resize(poolSize);
  cudaStream_t st = plan.stream;
  FKTB_CUDA(cudaMemcpyAsync(plan.dNearPool.get(), t.dNearPos.get(), static_cast<size_t>(t.nearTotal) * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, st));
  std::vector<uint32_t> ident(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) ident[static_cast<size_t>(i)] = static_cast<uint32_t>(i);
  FKTB_CUDA(cudaMemcpyAsync(plan.dNearPool.get() + t.nearTotal, ident.data(), ident.size() * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, st));
  if (!comp.empty())
    FKTB_CUDA(cudaMemcpyAsync(plan.dNearPool.get() + t.nearTotal + n, comp.data(), comp.size() * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, st));
  plan.blockTilesHost = std::move(tiles);
  plan.dBlockTiles.resize(std::max<size_t>(1, plan.blockTilesHost.size()));
  FKTB_CUDA(cudaMemcpyAsync(plan.dBlockTiles.get(), plan.blockTilesHost.data(),
                            plan.blockTilesHost.size() * sizeof(FktbBlockTile), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaStreamSynchronize(st));  // host vectors above are temporaries
  plan.symPairs = symPairs;
  plan.oneWayPairs = oneWay;
  plan.nearSym = true;
}

// The Gram-form symmetric kernel serves the smooth kernels without an r == 0
// select when every block's leaf passes the Gram bound (else the difference
// form below); FKTB_NEAR_SYM_DIFF=1 forces the difference form (A/B).
template <int KID>
bool launchSymGramK(const DevicePlan& plan, const double* yp, double* zp, double sc, double wf, int tiles,
                    cudaStream_t st) {
  const DeviceTree& t = *plan.tree;
  SymGArgs A{plan.n, t.pc.get(), plan.dNearPool.get(), plan.dBlockTiles.get(), yp, zp, expTableDevice(kNearExpBits),
             sc, wf, t.dCenter.get(), t.dLimit2.get(), kGramBoundSym / (sc * sc * (1.0 + t.theta * t.theta))};
  for (const FktbBlockTile& tl : plan.blockTilesHost) {
    volatile double limit = t.radius[static_cast<size_t>(tl.leaf)] / t.theta;
    if (!(limit * limit <= A.gramLimit2)) return false;
  }
  switch (plan.d) {
    case 2: near_sym_gram<KID, 2><<<tiles, 32, 0, st>>>(A); break;
    case 3: near_sym_gram<KID, 3><<<tiles, 32, 0, st>>>(A); break;
    case 5: near_sym_gram<KID, 5><<<tiles, 32, 0, st>>>(A); break;
    default: return false;
  }
  FKTB_CUDA(cudaGetLastError());
  return true;
}

bool launchNearSym(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t st) {
  if (!plan.nearSym || nrhs != 1 || plan.options.nearPrecision != 64) return false;
  const int tiles = static_cast<int>(plan.blockTilesHost.size());
  if (tiles == 0) return true;
  FktbKernelDesc kd;
  fillKernelDesc(plan.kernel, kd);
  if (plan.options.hasDiagonal) kd.diag = plan.options.diagonal;
  {
    double sc, wf;
    fastScales(kd, sc, wf);
    const char* e = std::getenv("FKTB_NEAR_SYM_DIFF");
    const bool forceDiff = e && e[0] == '1';
    if (!forceDiff && kd.diag == wf) {
      switch (kd.id) {
        case FKTB_KERNEL_MATERN32:
          if (launchSymGramK<FKTB_KERNEL_MATERN32>(plan, yp, zp, sc, wf, tiles, st)) return true;
          break;
        case FKTB_KERNEL_CAUCHY:
          if (launchSymGramK<FKTB_KERNEL_CAUCHY>(plan, yp, zp, sc, wf, tiles, st)) return true;
          break;
        case FKTB_KERNEL_RATIONAL_QUADRATIC:
          if (launchSymGramK<FKTB_KERNEL_RATIONAL_QUADRATIC>(plan, yp, zp, sc, wf, tiles, st)) return true;
          break;
        case FKTB_KERNEL_GAUSSIAN:
          if (launchSymGramK<FKTB_KERNEL_GAUSSIAN>(plan, yp, zp, sc, wf, tiles, st)) return true;
          break;
        default: break;
      }
    }
  }
  SymArgs A{plan.n, plan.tree->pc.get(), plan.dNearPool.get(), plan.dBlockTiles.get(), yp, zp, expTableDevice(kNearExpBits),
            1.0, 1.0, 0.0};
  fastScales(kd, A.sc, A.wf);
  A.diagCanon = kd.diag / A.wf;
  const bool smooth = kd.id != FKTB_KERNEL_INVERSE_R && kd.id != FKTB_KERNEL_INVERSE_R2;
  const bool sel = !(smooth && kd.diag == A.wf);
  switch (kd.id) {
    case FKTB_KERNEL_EXPONENTIAL: return launchSymK<FKTB_KERNEL_EXPONENTIAL>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_MATERN12: return launchSymK<FKTB_KERNEL_MATERN12>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_MATERN32: return launchSymK<FKTB_KERNEL_MATERN32>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_CAUCHY: return launchSymK<FKTB_KERNEL_CAUCHY>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return launchSymK<FKTB_KERNEL_RATIONAL_QUADRATIC>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_GAUSSIAN: return launchSymK<FKTB_KERNEL_GAUSSIAN>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_INVERSE_R: return launchSymK<FKTB_KERNEL_INVERSE_R>(A, plan.d, sel, tiles, st);
    case FKTB_KERNEL_INVERSE_R2: return launchSymK<FKTB_KERNEL_INVERSE_R2>(A, plan.d, sel, tiles, st);
    default: return false;
  }
}

}  // namespace fktb
