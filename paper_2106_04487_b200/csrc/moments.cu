// K4 source-to-multipole through monomial moments (see moments.hpp):
//   K4a p2m   : leaves, mu_a = sum_src y x'^a  (x' about the leaf center)
//   K4b m2m   : one launch per tree depth, bottom-up: parent mu from its two
//               children's mu shifted by delta = c_child - c_parent
//   K4c to_coef: per node with a far set, M = T mu (T carries Z_k nrm^2)
// Compile-time (d, p) shapes only; other shapes keep the direct S2M (far.cu).
#include <algorithm>

#include "device_math.cuh"
#include "plan.hpp"

namespace fktb {
namespace {

constexpr int kP2MThreads = 128;
constexpr int kRowPad = 1;  // odd per-lane row stride: conflict-free

constexpr int mono_count(int dims, int rem) {
  // binom(dims + rem, rem)
  long long b = 1;
  for (int i = 1; i <= rem; ++i) b = b * (dims + i) / i;
  return static_cast<int>(b);
}

// row[IDX + j] += prod * x^a over the monomials of dims [A, D) with degree
// <= REM, in the host enumeration order (MonomialBasis).
template <int D, int A, int REM, int IDX>
__device__ __forceinline__ void mono_accum(const double (&x)[D], double prod, double* row);

template <int D, int A, int REM, int IDX, int E>
__device__ __forceinline__ void mono_accum_e(const double (&x)[D], double prod, double* row) {
  if constexpr (E <= REM) {
    mono_accum<D, A + 1, REM - E, IDX>(x, prod, row);
    mono_accum_e<D, A, REM, IDX + mono_count(D - A - 1, REM - E), E + 1>(x, prod * x[A], row);
  }
}

template <int D, int A, int REM, int IDX>
__device__ __forceinline__ void mono_accum(const double (&x)[D], double prod, double* row) {
  if constexpr (A == D)
    row[IDX] += prod;
  else
    mono_accum_e<D, A, REM, IDX, 0>(x, prod, row);
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

template <int D, int P>
__global__ void __launch_bounds__(kP2MThreads, 1) p2m_kernel(const __grid_constant__ MomArgs A) {
  constexpr int C = mono_count(D, P);
  extern __shared__ double rows[];  // [threads][nrhs * C + pad]
  const int stride = C * A.nrhs + kRowPad;
  const FktbTile tile = A.tiles[blockIdx.x];
  const int leaf = tile.node;
  double* row = rows + static_cast<size_t>(threadIdx.x) * stride;
  for (int i = 0; i < stride; ++i) row[i] = 0.0;
  double c[D];
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = A.center[static_cast<size_t>(leaf) * D + a];
  for (int i = threadIdx.x; i < tile.count; i += kP2MThreads) {
    const int pos = static_cast<int>(tile.start) + i;
    double x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = A.pc[static_cast<size_t>(a) * A.n + pos] - c[a];
    for (int r = 0; r < A.nrhs; ++r) mono_accum<D, 0, P, 0>(x, A.yp[static_cast<size_t>(r) * A.n + pos], row + r * C);
  }
  __syncthreads();
  // column sums: warp w takes columns w, w+4, ...; lanes split the rows
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int col = warp; col < C * A.nrhs; col += kP2MThreads / 32) {
    double s = 0.0;
    for (int t = lane; t < kP2MThreads; t += 32) s += rows[static_cast<size_t>(t) * stride + col];
    s = warp_sum(s);
    if (lane == 0) {
      const int r = col / C, a = col % C;
      atomicAdd(A.mono + (static_cast<size_t>(r) * A.nodes + leaf) * C + a, s);
    }
  }
}

template <int D>
__global__ void m2m_kernel(const __grid_constant__ MomArgs A) {
  extern __shared__ double sm[];  // dpow[2][count], mu[2][nrhs][count]
  const int C = A.count;
  const int parent = A.levelNodes[blockIdx.x];
  const int kids[2] = {A.left[parent], A.right[parent]};
  double* dpow = sm;
  double* mu = sm + 2 * C;
  for (int i = threadIdx.x; i < 2 * C; i += blockDim.x) {
    const int ch = i / C, a = i % C;
    double v = 1.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      const double delta = A.center[static_cast<size_t>(kids[ch]) * D + q] - A.center[static_cast<size_t>(parent) * D + q];
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
      for (int e = A.off[a]; e < A.off[a + 1]; ++e) acc = fma(A.coef[e] * dp[A.g[e]], m[A.b[e]], acc);
    }
    A.mono[(static_cast<size_t>(r) * A.nodes + parent) * C + a] = acc;
  }
}

__global__ void to_coef_kernel(const __grid_constant__ MomArgs A) {
  extern __shared__ double mu[];  // [nrhs][count]
  const int C = A.count;
  const int node = A.farNodes[blockIdx.x];
  for (int i = threadIdx.x; i < A.nrhs * C; i += blockDim.x) {
    const int r = i / C, a = i % C;
    mu[i] = A.mono[(static_cast<size_t>(r) * A.nodes + node) * C + a];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < A.nrhs * A.P; i += blockDim.x) {
    const int r = i / A.P, c = i % A.P;
    const double* t = A.T + static_cast<size_t>(c) * C;
    const double* m = mu + static_cast<size_t>(r) * C;
    double acc = 0.0;
    for (int a = 0; a < C; ++a) acc = fma(t[a], m[a], acc);
    A.moments[(static_cast<size_t>(r) * A.nodes + node) * A.P + c] = acc;
  }
}

template <int D, int P>
void launchP2M(const MomArgs& A, int tiles, cudaStream_t st) {
  constexpr int C = mono_count(D, P);
  const size_t smem = static_cast<size_t>(kP2MThreads) * (C * A.nrhs + kRowPad) * sizeof(double);
  FKTB_CUDA(cudaFuncSetAttribute(p2m_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  p2m_kernel<D, P><<<tiles, kP2MThreads, smem, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

template <int D>
void launchM2M(const MomArgs& A, int parents, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(2 * A.count * (1 + A.nrhs)) * sizeof(double);
  if (smem > 48 * 1024)
    FKTB_CUDA(cudaFuncSetAttribute(m2m_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  m2m_kernel<D><<<parents, 128, smem, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

}  // namespace

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
  // K4a: per-lane rows must fit one CTA; chunk the right-hand sides.
  const size_t perRhs = static_cast<size_t>(kP2MThreads) * C * sizeof(double);
  const int chunk = std::max(1, static_cast<int>((200 * 1024) / perRhs));
  const int tiles = static_cast<int>(plan.p2mTilesHost.size());
  for (int r0 = 0; r0 < nrhs && tiles > 0; r0 += chunk) {
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
  for (int lv = static_cast<int>(plan.levelOff.size()) - 2; lv >= 0; --lv) {
    const int a0 = plan.levelOff[static_cast<size_t>(lv)], a1 = plan.levelOff[static_cast<size_t>(lv) + 1];
    if (a1 == a0) continue;
    MomArgs B = A;
    B.levelNodes = plan.dLevelNodes.get() + a0;
    switch (plan.d) {
      case 2: launchM2M<2>(B, a1 - a0, st); break;
      case 3: launchM2M<3>(B, a1 - a0, st); break;
      case 5: launchM2M<5>(B, a1 - a0, st); break;
      default: throw std::logic_error("monomial S2M: unsupported dimension");
    }
  }
  // K4c: node moments in the FKT basis.
  const int farNodes = static_cast<int>(plan.farNodesHost.size());
  if (farNodes > 0) {
    const size_t smem = static_cast<size_t>(nrhs) * C * sizeof(double);
    if (smem > 48 * 1024)
      FKTB_CUDA(cudaFuncSetAttribute(to_coef_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    to_coef_kernel<<<farNodes, 128, smem, st>>>(A);
    FKTB_CUDA(cudaGetLastError());
  }
}

}  // namespace fktb
