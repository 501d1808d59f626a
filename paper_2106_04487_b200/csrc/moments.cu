// K4 source-to-multipole through monomial moments (see moments.hpp):
//   K4a p2m   : leaves, mu_a = sum_src y x'^a  (x' about the leaf center).
//               Thread-owned (monomial, rhs) accumulators in registers;
//               sources staged in shared memory as per-axis power tables,
//               so each (source, item) is D broadcast loads + D multiplies.
//   K4b m2m   : one launch per tree depth, bottom-up: parent mu from its two
//               children's mu shifted by delta = c_child - c_parent
//   K4c to_coef: M = T mu for every node as one small GEMM (T carries
//               Z_k nrm^2 kappa^2; transposed copy for coalesced reads)
// Compile-time (d, p) shapes only; other shapes keep the direct S2M (far.cu).
#include <algorithm>
#include <cstdlib>

#include "device_math.cuh"
#include "plan.hpp"

namespace fktb {
namespace {


constexpr int mono_count(int dims, int rem) {
  // binom(dims + rem, rem)
  long long b = 1;
  for (int i = 1; i <= rem; ++i) b = b * (dims + i) / i;
  return static_cast<int>(b);
}

struct MomArgs {
  int n, nodes, count, nrhs, P;
  const double* pc;
  const double* center;
  const FktbTile* tiles;  // p2m: (leaf, count, start position)
  const double* yp;
  double* mono;           // [rhs][node][count]
  // m2m
  const int* levelNodes;
  const int* left;
  const int* right;
  const int* off;
  const int* b;
  const int* g;
  const double* coef;
  const int* exps;  // count x d
  // to_coef
  const int* farNodes;
  const double* T;  // P x count
  double* moments;  // [rhs][node][P]
};

constexpr int kP2MChunk = 64;     // sources staged per pass
constexpr int kP2MMaxThreads = 1024;

// One (rhs, monomial) accumulator per thread: item j = threadIdx.x,
// rhs j / C, monomial j % C (blockDim = C * nrhs rounded up to a warp).
template <int D, int P>
__global__ void __launch_bounds__(kP2MMaxThreads) p2m_regs(const __grid_constant__ MomArgs A) {
  constexpr int C = mono_count(D, P);
  constexpr int PW = P + 1;
  __shared__ double spw[kP2MChunk * D * PW];  // [src][axis][power]
  extern __shared__ double sw[];              // [src][rhs]
  const FktbTile tile = A.tiles[blockIdx.x];
  const int leaf = tile.node;
  const int j = threadIdx.x;
  const bool active = j < C * A.nrhs;
  const int a = active ? j % C : 0, rr = active ? j / C : 0;
  int off[D];
#pragma unroll
  for (int q = 0; q < D; ++q) off[q] = q * PW + A.exps[a * D + q];
  double acc = 0.0;
  double c[D];
#pragma unroll
  for (int q = 0; q < D; ++q) c[q] = A.center[static_cast<size_t>(leaf) * D + q];
  for (int s0 = 0; s0 < tile.count; s0 += kP2MChunk) {
    const int cn = min(kP2MChunk, tile.count - s0);
    __syncthreads();
    for (int t = threadIdx.x; t < cn * D; t += blockDim.x) {
      const int s = t / D, q = t % D;
      const int pos = static_cast<int>(tile.start) + s0 + s;
      const double x = A.pc[static_cast<size_t>(q) * A.n + pos] - c[q];
      double* row = spw + (s * D + q) * PW;
      double v = 1.0;
      row[0] = 1.0;
#pragma unroll
      for (int e = 1; e <= P; ++e) {
        v *= x;
        row[e] = v;
      }
    }
    for (int t = threadIdx.x; t < cn * A.nrhs; t += blockDim.x) {
      const int s = t / A.nrhs, r = t % A.nrhs;
      sw[t] = A.yp[static_cast<size_t>(r) * A.n + tile.start + s0 + s];
    }
    __syncthreads();
    if (active) {
#pragma unroll 4
      for (int s = 0; s < cn; ++s) {
        const double* pw = spw + s * D * PW;
        double m = sw[s * A.nrhs + rr];
#pragma unroll
        for (int q = 0; q < D - 1; ++q) m *= pw[off[q]];
        acc = fma(m, pw[off[D - 1]], acc);
      }
    }
  }
  if (active) atomicAdd(A.mono + (static_cast<size_t>(rr) * A.nodes + leaf) * C + a, acc);
}

// Multi-RHS P2M: a warp per source stream (kP2MGroups warps split the tile's
// sources), lane l owning monomials l, l + 32, ... for RB right-hand sides in
// registers. Each (source, monomial) product x'^a is formed once (D broadcast
// power loads) and feeds RB FMAs against the source's RB weights (RB/2
// broadcast LDS.128), instead of RB x (D + 1 loads + D FP64 ops) with one
// (rhs, monomial) per thread (p2m_regs). The groups' partial sums are reduced
// in shared memory, one atomic per (rhs, monomial) per tile.
constexpr int kP2MGroups = 8;
template <int D, int P, int RB>
__global__ void __launch_bounds__(32 * kP2MGroups) p2m_multi(const __grid_constant__ MomArgs A) {
  constexpr int C = mono_count(D, P);
  constexpr int PW = P + 1;
  constexpr int AM = (C + 31) / 32;  // monomials per lane
  constexpr int CH = 64;             // sources staged per pass
  __shared__ double spw[CH * D * PW];                // [src][axis][power]
  __shared__ __align__(16) double sw[CH * RB];       // [src][rhs]
  __shared__ double sred[AM * RB * 32];              // the groups' partial sums, reduced in turn
  const FktbTile tile = A.tiles[blockIdx.x];
  const int leaf = tile.node;
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  int off[AM][D];
  bool own[AM];
#pragma unroll
  for (int m = 0; m < AM; ++m) {
    const int a = lane + 32 * m;
    own[m] = a < C;
#pragma unroll
    for (int q = 0; q < D; ++q) off[m][q] = q * PW + (own[m] ? A.exps[a * D + q] : 0);
  }
  double c[D];
#pragma unroll
  for (int q = 0; q < D; ++q) c[q] = A.center[static_cast<size_t>(leaf) * D + q];
  for (int r0 = 0; r0 < A.nrhs; r0 += RB) {
    double acc[AM][RB];
#pragma unroll
    for (int m = 0; m < AM; ++m)
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[m][r] = 0.0;
    for (int s0 = 0; s0 < tile.count; s0 += CH) {
      const int cn = min(CH, tile.count - s0);
      __syncthreads();
      for (int t = threadIdx.x; t < cn * D; t += blockDim.x) {
        const int s = t / D, q = t % D;
        const int pos = static_cast<int>(tile.start) + s0 + s;
        const double x = A.pc[static_cast<size_t>(q) * A.n + pos] - c[q];
        double* row = spw + (s * D + q) * PW;
        double v = 1.0;
        row[0] = 1.0;
#pragma unroll
        for (int e = 1; e <= P; ++e) {
          v *= x;
          row[e] = v;
        }
      }
      for (int t = threadIdx.x; t < cn * RB; t += blockDim.x) {
        const int s = t / RB, r = t % RB;
        sw[t] = A.yp[static_cast<size_t>(r0 + r) * A.n + tile.start + s0 + s];
      }
      __syncthreads();
      for (int s = grp; s < cn; s += kP2MGroups) {
        const double* pw = spw + s * D * PW;
        double w[RB];
        if constexpr (RB == 1) {
          w[0] = sw[s];
        } else {
#pragma unroll
          for (int r = 0; r < RB; r += 2) {
            const double2 v = *reinterpret_cast<const double2*>(sw + s * RB + r);
            w[r] = v.x;
            w[r + 1] = v.y;
          }
        }
#pragma unroll
        for (int m = 0; m < AM; ++m) {
          double mono = pw[off[m][0]];
#pragma unroll
          for (int q = 1; q < D; ++q) mono *= pw[off[m][q]];
#pragma unroll
          for (int r = 0; r < RB; ++r) acc[m][r] = fma(mono, w[r], acc[m][r]);
        }
      }
    }
    // reduce the groups' partial sums in turn (fixed order), then one atomic
    // per (rhs, monomial)
    for (int g2 = 0; g2 < kP2MGroups; ++g2) {
      __syncthreads();
      if (grp == g2)
#pragma unroll
        for (int m = 0; m < AM; ++m)
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            double& dst = sred[(m * RB + r) * 32 + lane];
            dst = g2 == 0 ? acc[m][r] : dst + acc[m][r];
          }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < AM * RB * 32; i += blockDim.x) {
      const int l = i & 31, mr = i >> 5, m = mr / RB, r = mr % RB;
      const int a = l + 32 * m;
      if (a < C) atomicAdd(A.mono + (static_cast<size_t>(r0 + r) * A.nodes + leaf) * C + a, sred[i]);
    }
  }
}

// Shift tables (CSR over the output monomial) staged in shared memory once
// per CTA; each CTA then walks parents blockIdx.x, blockIdx.x + gridDim.x, ...
template <int D>
__global__ void m2m_kernel(const __grid_constant__ MomArgs A, int parents, int entries) {
  extern __shared__ double sm[];  // coef[E] | dpow[2][C] | mu[2][nrhs][C] | off[C+1] b[E] g[E] (ints)
  const int C = A.count;
  double* scoef = sm;
  double* dpow = scoef + entries;
  double* mu = dpow + 2 * C;
  int* soff = reinterpret_cast<int*>(mu + 2 * A.nrhs * C);
  int* sb = soff + C + 1;
  int* sg = sb + entries;
  for (int i = threadIdx.x; i < entries; i += blockDim.x) {
    scoef[i] = A.coef[i];
    sb[i] = A.b[i];
    sg[i] = A.g[i];
  }
  for (int i = threadIdx.x; i <= C; i += blockDim.x) soff[i] = A.off[i];
  for (int pi = blockIdx.x; pi < parents; pi += gridDim.x) {
    const int parent = A.levelNodes[pi];
    const int kids[2] = {A.left[parent], A.right[parent]};
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * C; i += blockDim.x) {
      const int ch = i / C, a = i % C;
      double v = 1.0;
#pragma unroll
      for (int q = 0; q < D; ++q) {
        const double delta =
            A.center[static_cast<size_t>(kids[ch]) * D + q] - A.center[static_cast<size_t>(parent) * D + q];
        for (int e = 0; e < A.exps[a * D + q]; ++e) v *= delta;
      }
      dpow[i] = v;
    }
    for (int i = threadIdx.x; i < 2 * A.nrhs * C; i += blockDim.x) {
      const int ch = i / (A.nrhs * C), rem = i % (A.nrhs * C), r = rem / C, a = rem % C;
      mu[i] = A.mono[(static_cast<size_t>(r) * A.nodes + kids[ch]) * C + a];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < A.nrhs * C; i += blockDim.x) {
      const int r = i / C, a = i % C;
      double acc = 0.0;
      for (int ch = 0; ch < 2; ++ch) {
        const double* dp = dpow + ch * C;
        const double* m = mu + (static_cast<size_t>(ch) * A.nrhs + r) * C;
        for (int e = soff[a]; e < soff[a + 1]; ++e) acc = fma(scoef[e] * dp[sg[e]], m[sb[e]], acc);
      }
      A.mono[(static_cast<size_t>(r) * A.nodes + parent) * C + a] = acc;
    }
  }
}

// The narrow top of the tree in one launch: CTA per (node b, frontier node f)
// adds Shift(c_f - c_b) mu_f into mu_b (atomics; mu_b starts at zero from the
// S2M memset). The monomial shift is the M2M's with an arbitrary delta, so a
// composite shift over several levels is exact up to rounding:
// mu_b[a] = sum_f sum_{e in CSR(a)} coef_e delta_f^g_e mu_f[b_e].
template <int D>
__global__ void m2m_pairs(const __grid_constant__ MomArgs A, const int* pairs, int entries) {
  extern __shared__ double sm[];  // coef[E] | dpow[C] | mu[nrhs][C] | off[C+1] b[E] g[E] (ints)
  const int C = A.count;
  double* scoef = sm;
  double* dpow = scoef + entries;
  double* mu = dpow + C;
  int* soff = reinterpret_cast<int*>(mu + A.nrhs * C);
  int* sb = soff + C + 1;
  int* sg = sb + entries;
  const int b = pairs[2 * blockIdx.x], f = pairs[2 * blockIdx.x + 1];
  for (int i = threadIdx.x; i < entries; i += blockDim.x) {
    scoef[i] = A.coef[i];
    sb[i] = A.b[i];
    sg[i] = A.g[i];
  }
  for (int i = threadIdx.x; i <= C; i += blockDim.x) soff[i] = A.off[i];
  for (int a = threadIdx.x; a < C; a += blockDim.x) {
    double v = 1.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      const double delta = A.center[static_cast<size_t>(f) * D + q] - A.center[static_cast<size_t>(b) * D + q];
      for (int e = 0; e < A.exps[a * D + q]; ++e) v *= delta;
    }
    dpow[a] = v;
  }
  for (int i = threadIdx.x; i < A.nrhs * C; i += blockDim.x) {
    const int r = i / C, a = i % C;
    mu[i] = A.mono[(static_cast<size_t>(r) * A.nodes + f) * C + a];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < A.nrhs * C; i += blockDim.x) {
    const int r = i / C, a = i % C;
    const double* m = mu + static_cast<size_t>(r) * C;
    double acc = 0.0;
    for (int e = soff[a]; e < soff[a + 1]; ++e) acc = fma(scoef[e] * dpow[sg[e]], m[sb[e]], acc);
    atomicAdd(A.mono + (static_cast<size_t>(r) * A.nodes + b) * C + a, acc);
  }
}

// Node moments in the FKT basis for every (rhs, node) row: out[R][P] =
// mono[R][C] * TT[C][P] -- a small GEMM, 32 rows per CTA staged in shared
// memory (even row stride: each thread reads two monomials of a row with one
// broadcast LDS.128), TT columns read coalesced (L1/L2 resident).
constexpr int kTcRows = 32;
// Threads cover (row group, output column): with P < blockDim the 32 staged
// rows split into G = blockDim / P groups (cfg5: P = 28 -> 4 groups of 8 rows,
// 112 of 128 threads busy instead of 28). T columns are prefetched four
// monomials ahead (the loads were the loop's latency).
template <int RPT>
__device__ __forceinline__ void to_coef_rows(const double* smu, const double* TT, double* out, int r0, int rows,
                                             int row0, int c, int C, int CS, int P) {
  double acc[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) acc[i] = 0.0;
  int a = 0;
  for (; a + 3 < C; a += 4) {
    double t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = TT[static_cast<size_t>(a + j) * P + c];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const double2 m0 = *reinterpret_cast<const double2*>(smu + (row0 + i) * CS + a);
      const double2 m1 = *reinterpret_cast<const double2*>(smu + (row0 + i) * CS + a + 2);
      acc[i] = fma(t[3], m1.y, fma(t[2], m1.x, fma(t[1], m0.y, fma(t[0], m0.x, acc[i]))));
    }
  }
  for (; a < C; ++a) {
    const double t0 = TT[static_cast<size_t>(a) * P + c];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i] = fma(t0, smu[(row0 + i) * CS + a], acc[i]);
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i)
    if (row0 + i < rows) out[static_cast<size_t>(r0 + row0 + i) * P + c] = acc[i];
}

__global__ void __launch_bounds__(128) to_coef_gemm(const double* mono, const double* TT, double* out, int R, int C,
                                                   int P) {
  extern __shared__ __align__(16) double smu[];  // [kTcRows][CS], CS = C rounded up to even
  const int CS = (C + 1) & ~1;
  const int r0 = blockIdx.x * kTcRows;
  const int rows = min(kTcRows, R - r0);
  for (int i = threadIdx.x; i < kTcRows * CS; i += blockDim.x) {
    const int rr = i / CS, a = i % CS;
    smu[i] = rr < rows && a < C ? mono[static_cast<size_t>(r0 + rr) * C + a] : 0.0;
  }
  __syncthreads();
  const int T = static_cast<int>(blockDim.x);
  if (4 * P <= T) {  // four row groups of 8
    const int g = threadIdx.x / P, c = threadIdx.x - g * P;
    if (g < 4) to_coef_rows<8>(smu, TT, out, r0, rows, 8 * g, c, C, CS, P);
  } else if (2 * P <= T) {  // two row groups of 16
    const int g = threadIdx.x / P, c = threadIdx.x - g * P;
    if (g < 2) to_coef_rows<16>(smu, TT, out, r0, rows, 16 * g, c, C, CS, P);
  } else {
    for (int c = threadIdx.x; c < P; c += T) to_coef_rows<kTcRows>(smu, TT, out, r0, rows, 0, c, C, CS, P);
  }
}

// Multi-RHS P2M block size: RB right-hand sides per pass with AM x RB <= 48
// register accumulators per lane (0: not applicable, keep p2m_regs).
template <int D, int P>
constexpr int p2mMultiBlock() {
  constexpr int AM = (mono_count(D, P) + 31) / 32;
  return AM * 16 <= 48 ? 16 : (AM * 8 <= 48 ? 8 : 0);
}

template <int D, int P>
void launchP2M(const MomArgs& A, int tiles, cudaStream_t st) {
  constexpr int C = mono_count(D, P);
  const int threads = std::min(kP2MMaxThreads, (C * A.nrhs + 31) / 32 * 32);
  const size_t smem = static_cast<size_t>(kP2MChunk) * A.nrhs * sizeof(double);
  p2m_regs<D, P><<<tiles, threads, smem, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

template <int D, int P>
bool launchP2MMulti(const MomArgs& A, int tiles, cudaStream_t st) {
  constexpr int RB = p2mMultiBlock<D, P>();
  if constexpr (RB == 0) {
    return false;
  } else {
    if (A.nrhs % RB != 0) return false;
    p2m_multi<D, P, RB><<<tiles, 32 * kP2MGroups, 0, st>>>(A);
    FKTB_CUDA(cudaGetLastError());
    return true;
  }
}



template <int D>
void launchM2MPairs(const MomArgs& A, const int* pairs, int npairs, int entries, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024)
    FKTB_CUDA(cudaFuncSetAttribute(m2m_pairs<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  m2m_pairs<D><<<npairs, 256, smem, st>>>(A, pairs, entries);
  FKTB_CUDA(cudaGetLastError());
}

template <int D>
void launchM2M(const MomArgs& A, int parents, int entries, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(entries + 2 * A.count * (1 + A.nrhs)) * sizeof(double) +
                      static_cast<size_t>(A.count + 1 + 2 * entries) * sizeof(int);
  if (smem > 48 * 1024)
    FKTB_CUDA(cudaFuncSetAttribute(m2m_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int grid = std::min(parents, 148 * 2);
  m2m_kernel<D><<<grid, 256, smem, st>>>(A, parents, entries);
  FKTB_CUDA(cudaGetLastError());
}

}  // namespace

// P2M launches of one multiply (kernelLaunches): one p2m_multi launch when the
// RHS-blocked path applies, else one p2m_regs launch per RHS chunk.
int p2mLaunches(int d, int p, int count, int nrhs) {
  int rb = 0;
  switch (d * 100 + p) {
    case 206: rb = p2mMultiBlock<2, 6>(); break;
    case 304: rb = p2mMultiBlock<3, 4>(); break;
    case 306: rb = p2mMultiBlock<3, 6>(); break;
    case 308: rb = p2mMultiBlock<3, 8>(); break;
    case 504: rb = p2mMultiBlock<5, 4>(); break;
    default: break;
  }
  if (rb > 0 && nrhs >= 8 && nrhs % rb == 0) return 1;
  const int chunk = std::max(1, kP2MMaxThreads / count);
  return (nrhs + chunk - 1) / chunk;
}

bool momentsSupported(int d, int p) {
  switch (d * 100 + p) {
    case 206:
    case 304:
    case 306:
    case 308:
    case 504: return true;
    default: return false;
  }
}

void launchS2MMoments(const DevicePlan& plan, const double* yp, double* moments, int nrhs, cudaStream_t st) {
  const DeviceTree& t = *plan.tree;
  const int C = plan.monoCount;
  MomArgs A{};
  A.n = t.n;
  A.nodes = t.nodes;
  A.count = C;
  A.P = plan.P;
  A.pc = t.pc.get();
  A.center = t.dCenter.get();
  A.tiles = plan.dP2mTiles.get();
  A.mono = plan.dMono.get();
  A.left = t.dLeft.get();
  A.right = t.dRight.get();
  A.off = plan.dShiftOff.get();
  A.b = plan.dShiftB.get();
  A.g = plan.dShiftG.get();
  A.coef = plan.dShiftCoef.get();
  A.exps = plan.dMonoExps.get();
  A.farNodes = plan.dFarNodes.get();
  A.T = plan.dMomT.get();
  A.moments = moments;
  FKTB_CUDA(cudaMemsetAsync(plan.dMono.get(), 0, static_cast<size_t>(t.nodes) * C * nrhs * sizeof(double), st));
  // K4a: one accumulator per thread, at most kP2MMaxThreads per CTA; chunk the
  // right-hand sides to fit.
  const int chunk = std::max(1, kP2MMaxThreads / C);
  const int tiles = static_cast<int>(plan.p2mTilesHost.size());
  // many right-hand sides: RHS-blocked p2m_multi (monomial formed once per
  // source and reused for the block)
  auto multi = [&]() -> bool {
    if (tiles == 0 || nrhs < 8) return false;
    MomArgs B = A;
    B.nrhs = nrhs;
    B.yp = yp;
    switch (plan.d * 100 + plan.options.p) {
      case 206: return launchP2MMulti<2, 6>(B, tiles, st);
      case 304: return launchP2MMulti<3, 4>(B, tiles, st);
      case 306: return launchP2MMulti<3, 6>(B, tiles, st);
      case 308: return launchP2MMulti<3, 8>(B, tiles, st);
      case 504: return launchP2MMulti<5, 4>(B, tiles, st);
      default: return false;
    }
  };
  const bool didMulti = multi();
  for (int r0 = 0; r0 < nrhs && tiles > 0 && !didMulti; r0 += chunk) {
    MomArgs B = A;
    B.nrhs = std::min(chunk, nrhs - r0);
    B.yp = yp + static_cast<size_t>(r0) * t.n;
    B.mono = plan.dMono.get() + static_cast<size_t>(r0) * t.nodes * C;
    switch (plan.d * 100 + plan.options.p) {
      case 206: launchP2M<2, 6>(B, tiles, st); break;
      case 304: launchP2M<3, 4>(B, tiles, st); break;
      case 306: launchP2M<3, 6>(B, tiles, st); break;
      case 308: launchP2M<3, 8>(B, tiles, st); break;
      case 504: launchP2M<5, 4>(B, tiles, st); break;
      default: throw std::logic_error("monomial S2M: unsupported shape");
    }
  }
  // K4b: bottom-up shifts, deepest internal level first.
  A.nrhs = nrhs;
  A.yp = yp;
  for (int lv = static_cast<int>(plan.levelOff.size()) - 2; lv >= plan.m2mTop; --lv) {
    const int a0 = plan.levelOff[static_cast<size_t>(lv)], a1 = plan.levelOff[static_cast<size_t>(lv) + 1];
    if (a1 == a0) continue;
    MomArgs B = A;
    B.levelNodes = plan.dLevelNodes.get() + a0;
    switch (plan.d) {
      case 2: launchM2M<2>(B, a1 - a0, plan.shiftEntries, st); break;
      case 3: launchM2M<3>(B, a1 - a0, plan.shiftEntries, st); break;
      case 5: launchM2M<5>(B, a1 - a0, plan.shiftEntries, st); break;
      default: throw std::logic_error("monomial S2M: unsupported dimension");
    }
  }
  if (plan.topPairs > 0) {  // the narrow top levels from their frontier, one launch
    MomArgs B = A;
    const size_t smem = static_cast<size_t>(plan.shiftEntries + C * (1 + nrhs)) * sizeof(double) +
                        static_cast<size_t>(C + 1 + 2 * plan.shiftEntries) * sizeof(int);
    switch (plan.d) {
      case 2: launchM2MPairs<2>(B, plan.dTopPairs.get(), plan.topPairs, plan.shiftEntries, smem, st); break;
      case 3: launchM2MPairs<3>(B, plan.dTopPairs.get(), plan.topPairs, plan.shiftEntries, smem, st); break;
      case 5: launchM2MPairs<5>(B, plan.dTopPairs.get(), plan.topPairs, plan.shiftEntries, smem, st); break;
      default: throw std::logic_error("monomial S2M: unsupported dimension");
    }
  }
  // K4c: node moments in the FKT basis, every (rhs, node) row at once.
  if (!plan.farNodesHost.empty()) {
    const int R = nrhs * t.nodes;
    const size_t smem = static_cast<size_t>(kTcRows) * ((C + 1) & ~1) * sizeof(double);
    if (smem > 48 * 1024)
      FKTB_CUDA(cudaFuncSetAttribute(to_coef_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // single-RHS passes of plans with a Cartesian M2T: its coefficients
    const bool cart = cartPass(plan, nrhs);
    to_coef_gemm<<<(R + kTcRows - 1) / kTcRows, 128, smem, st>>>(
        plan.dMono.get(), cart ? plan.dCartTT.get() : plan.dMomTT.get(), moments, R, C, momentStride(plan, nrhs));
    FKTB_CUDA(cudaGetLastError());
  }
}

}  // namespace fktb
