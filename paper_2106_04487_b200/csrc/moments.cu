// K4 source-to-multipole through monomial moments (see moments.hpp):
//   K4a p2m   : leaves, mu_a = sum_src y x'^a  (x' about the leaf center).
//               Thread-owned (monomial, rhs) accumulators in registers;
//               sources staged in shared memory as per-axis power tables,
//               so each (source, item) is D broadcast loads + D multiplies.
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

constexpr int kP2MChunk = 64;  // sources staged per pass

// ITEMS accumulators per thread: items j = threadIdx.x + i * kP2MThreads,
// item j = (rhs j / C, monomial j % C).
template <int D, int P, int ITEMS>
__global__ void __launch_bounds__(kP2MThreads) p2m_regs(const __grid_constant__ MomArgs A) {
  constexpr int C = mono_count(D, P);
  constexpr int PW = P + 1;
  __shared__ double spw[kP2MChunk * D * PW];  // [src][axis][power]
  extern __shared__ double sw[];              // [src][rhs]
  const FktbTile tile = A.tiles[blockIdx.x];
  const int leaf = tile.node;
  const int items = C * A.nrhs;
  int off[ITEMS][D];  // offsets into one source's power table, per axis
  int rr[ITEMS];
  double acc[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int j = threadIdx.x + i * kP2MThreads;
    const int a = j < items ? j % C : 0;
    rr[i] = j < items ? j / C : -1;
#pragma unroll
    for (int q = 0; q < D; ++q) off[i][q] = q * PW + A.exps[a * D + q];
    acc[i] = 0.0;
  }
  double c[D];
#pragma unroll
  for (int q = 0; q < D; ++q) c[q] = A.center[static_cast<size_t>(leaf) * D + q];
  for (int s0 = 0; s0 < tile.count; s0 += kP2MChunk) {
    const int cn = min(kP2MChunk, tile.count - s0);
    __syncthreads();
    for (int t = threadIdx.x; t < cn * D; t += kP2MThreads) {
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
    for (int t = threadIdx.x; t < cn * A.nrhs; t += kP2MThreads) {
      const int s = t / A.nrhs, r = t % A.nrhs;
      sw[t] = A.yp[static_cast<size_t>(r) * A.n + tile.start + s0 + s];
    }
    __syncthreads();
    for (int s = 0; s < cn; ++s) {
      const double* pw = spw + s * D * PW;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (rr[i] < 0) continue;
        double m = sw[s * A.nrhs + rr[i]];
#pragma unroll
        for (int q = 0; q < D - 1; ++q) m *= pw[off[i][q]];
        acc[i] = fma(m, pw[off[i][D - 1]], acc[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (rr[i] < 0) continue;
    const int j = threadIdx.x + i * kP2MThreads;
    atomicAdd(A.mono + (static_cast<size_t>(rr[i]) * A.nodes + leaf) * C + j % C, acc[i]);
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

constexpr int kP2MMaxItems = 8;

template <int D, int P>
void launchP2M(const MomArgs& A, int tiles, cudaStream_t st) {
  constexpr int C = mono_count(D, P);
  const int per = (C * A.nrhs + kP2MThreads - 1) / kP2MThreads;
  const size_t smem = static_cast<size_t>(kP2MChunk) * A.nrhs * sizeof(double);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      FKTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<tiles, kP2MThreads, smem, st>>>(A);
  };
  if (per <= 1)
    go(p2m_regs<D, P, 1>);
  else if (per <= 2)
    go(p2m_regs<D, P, 2>);
  else if (per <= 4)
    go(p2m_regs<D, P, 4>);
  else
    go(p2m_regs<D, P, kP2MMaxItems>);
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
  // K4a: at most kP2MMaxItems register accumulators per thread; chunk the
  // right-hand sides to fit.
  const int chunk = std::max(1, kP2MMaxItems * kP2MThreads / C);
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
