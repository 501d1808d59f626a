// K3 near field, FP32 fast mode (north star: "accumulates z in fp64, plus an
// fp32 fast mode"). Opt-in per plan (FktOptions nearPrecision = 32); the far
// field stays FP64.
//
// Coordinates are taken relative to the leaf's center and scaled by the
// kernel length scale in FP64, then rounded to FP32, so the pair differences
// keep ~1e-7 relative accuracy regardless of where the leaf sits. The kernel
// is evaluated with SFU intrinsics (ex2/rsqrt/rcp approx) on the FP32 pipe,
// each target's contribution from one leaf is summed in FP32 (<= a few
// hundred terms) and added to z in FP64. Expected z error ~1e-6 relative;
// tests/test_gpu_fp32.py pins it against the FP64 path.
#include <cmath>

#include "fastmath.cuh"
#include "plan.hpp"

namespace fktb {
namespace {

constexpr int kChunk32 = 512;

template <int KID>
struct Kernel32 {
  static constexpr bool supported =
      KID == FKTB_KERNEL_MATERN32 || KID == FKTB_KERNEL_MATERN12 || KID == FKTB_KERNEL_EXPONENTIAL ||
      KID == FKTB_KERNEL_CAUCHY || KID == FKTB_KERNEL_RATIONAL_QUADRATIC || KID == FKTB_KERNEL_GAUSSIAN ||
      KID == FKTB_KERNEL_INVERSE_R || KID == FKTB_KERNEL_INVERSE_R2;
  // canonical K at scaled squared distance q > 0
  __device__ static __forceinline__ float eval(float q) {
    if constexpr (KID == FKTB_KERNEL_MATERN32) {
      const float u = q * rsqrtf(q);
      const float e = __expf(-u);
      return fmaf(u, e, e);
    } else if constexpr (KID == FKTB_KERNEL_MATERN12 || KID == FKTB_KERNEL_EXPONENTIAL) {
      return __expf(-(q * rsqrtf(q)));
    } else if constexpr (KID == FKTB_KERNEL_CAUCHY) {
      return __frcp_rn(1.0f + q);
    } else if constexpr (KID == FKTB_KERNEL_RATIONAL_QUADRATIC) {
      return rsqrtf(1.0f + q);
    } else if constexpr (KID == FKTB_KERNEL_GAUSSIAN) {
      return __expf(-q);
    } else if constexpr (KID == FKTB_KERNEL_INVERSE_R) {
      return rsqrtf(q);
    } else {
      return __frcp_rn(q);
    }
  }
};

struct Args32 {
  int n, d, nrhs;
  const double* pc;
  const double* center;
  const uint32_t* begin;
  const uint32_t* end;
  const FktbTile* tiles;
  const uint32_t* nearPos;
  const double* yp;
  ZOut out;
  double sc, wf;
  float diagCanon;
  int sel;
};

constexpr float kQBias32 = 1e-30f;

template <int KID, int D, bool SEL, int THREADS, int TPT, int R>
__global__ void __launch_bounds__(THREADS) near_fp32(const __grid_constant__ Args32 A) {
  constexpr int SP = (D + R + 3) / 4 * 4;  // AoS float stride, 16-byte aligned
  __shared__ __align__(16) float ss[kChunk32 * SP];
  const FktbTile tile = A.tiles[blockIdx.x];
  const int leaf = tile.node;
  const int sb = static_cast<int>(A.begin[leaf]), se = static_cast<int>(A.end[leaf]);
  const int n = A.n;
  double c[D];
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = A.center[static_cast<size_t>(leaf) * D + a];
  int tpos[TPT];
  float tx[TPT][D];
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    const int idx = threadIdx.x + i * THREADS;
    tpos[i] = idx < tile.count ? static_cast<int>(A.nearPos[tile.start + idx]) : -1;
    const int p = tpos[i] >= 0 ? tpos[i] : 0;
#pragma unroll
    for (int a = 0; a < D; ++a) tx[i][a] = static_cast<float>((A.pc[static_cast<size_t>(a) * n + p] - c[a]) * A.sc);
  }
  for (int r0 = 0; r0 < A.nrhs; r0 += R) {
    float acc[TPT][R];
    double accd[TPT][R];
#pragma unroll
    for (int i = 0; i < TPT; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) accd[i][r] = 0.0;
    for (int cs = sb; cs < se; cs += kChunk32) {
      const int cn = min(kChunk32, se - cs);
      __syncthreads();
      for (int s = threadIdx.x; s < cn; s += THREADS) {
#pragma unroll
        for (int a = 0; a < D; ++a)
          ss[s * SP + a] = static_cast<float>((A.pc[static_cast<size_t>(a) * n + cs + s] - c[a]) * A.sc);
#pragma unroll
        for (int r = 0; r < R; ++r)
          ss[s * SP + D + r] = static_cast<float>(A.yp[static_cast<size_t>(r0 + r) * n + cs + s] * A.wf);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < TPT; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[i][r] = 0.0f;
#pragma unroll 4
      for (int s = 0; s < cn; ++s) {
        float src[SP];
#pragma unroll
        for (int q = 0; q < SP; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(&ss[s * SP + q]);
          src[q] = v.x;
          src[q + 1] = v.y;
          src[q + 2] = v.z;
          src[q + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < TPT; ++i) {
          const float d0 = tx[i][0] - src[0];
          float q = fmaf(d0, d0, kQBias32);
#pragma unroll
          for (int a = 1; a < D; ++a) {
            const float da = tx[i][a] - src[a];
            q = fmaf(da, da, q);
          }
          float kv = Kernel32<KID>::eval(q);
          if constexpr (SEL) kv = q == kQBias32 ? A.diagCanon : kv;
#pragma unroll
          for (int r = 0; r < R; ++r) acc[i][r] = fmaf(kv, src[D + r], acc[i][r]);
        }
      }
#pragma unroll
      for (int i = 0; i < TPT; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r) accd[i][r] += static_cast<double>(acc[i][r]);
    }
#pragma unroll
    for (int i = 0; i < TPT; ++i)
      if (tpos[i] >= 0)
#pragma unroll
        for (int r = 0; r < R; ++r) A.out.add(r0 + r, tile.start + threadIdx.x + i * THREADS, tpos[i], accd[i][r]);
  }
}

template <int KID, int D, bool SEL>
void launch32(const Args32& A, int tiles, cudaStream_t st) {
  if (A.nrhs % 16 == 0)
    near_fp32<KID, D, SEL, 256, 1, 16><<<tiles, 256, 0, st>>>(A);
  else if (A.nrhs % 4 == 0)
    near_fp32<KID, D, SEL, 128, 2, 4><<<tiles, 128, 0, st>>>(A);
  else
    near_fp32<KID, D, SEL, 64, 4, 1><<<tiles, 64, 0, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

template <int KID>
bool launchK32(const Args32& A, int tiles, cudaStream_t st) {
  if constexpr (!Kernel32<KID>::supported) {
    return false;
  } else {
    auto go = [&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (A.sel)
        launch32<KID, D, true>(A, tiles, st);
      else
        launch32<KID, D, false>(A, tiles, st);
    };
    switch (A.d) {
      case 2: go(std::integral_constant<int, 2>{}); return true;
      case 3: go(std::integral_constant<int, 3>{}); return true;
      case 5: go(std::integral_constant<int, 5>{}); return true;
      default: return false;
    }
  }
}

}  // namespace

// Returns false when (kernel, d) has no FP32 variant (the caller then runs
// the FP64 near field).
bool launchNear32(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t st) {
  const int tiles = static_cast<int>(plan.nearTilesHost.size());
  if (tiles == 0) return true;
  const DeviceTree& t = *plan.tree;
  FktbKernelDesc kd;
  fillKernelDesc(plan.kernel, kd);
  if (plan.options.hasDiagonal) kd.diag = plan.options.diagonal;
  Args32 A{t.n, t.d, nrhs, t.pc.get(), t.dCenter.get(), t.dBegin.get(), t.dEnd.get(), plan.dNearTiles.get(),
           t.dNearPos.get(), yp, zoutFor(plan, zp, nrhs, false), 1.0, 1.0, 0.0f, 0};
  switch (kd.id) {
    case FKTB_KERNEL_MATERN32: A.sc = kd.a; A.wf = kd.s2; break;
    case FKTB_KERNEL_MATERN12: A.sc = 1.0 / kd.rho; A.wf = kd.s2; break;
    case FKTB_KERNEL_CAUCHY:
    case FKTB_KERNEL_RATIONAL_QUADRATIC: A.sc = std::sqrt(kd.is2); break;
    default: break;
  }
  const bool smooth = kd.id != FKTB_KERNEL_INVERSE_R && kd.id != FKTB_KERNEL_INVERSE_R2;
  A.sel = !(smooth && kd.diag == A.wf);
  A.diagCanon = static_cast<float>(kd.diag / A.wf);
  switch (kd.id) {
    case FKTB_KERNEL_EXPONENTIAL: return launchK32<FKTB_KERNEL_EXPONENTIAL>(A, tiles, st);
    case FKTB_KERNEL_MATERN12: return launchK32<FKTB_KERNEL_MATERN12>(A, tiles, st);
    case FKTB_KERNEL_MATERN32: return launchK32<FKTB_KERNEL_MATERN32>(A, tiles, st);
    case FKTB_KERNEL_CAUCHY: return launchK32<FKTB_KERNEL_CAUCHY>(A, tiles, st);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return launchK32<FKTB_KERNEL_RATIONAL_QUADRATIC>(A, tiles, st);
    case FKTB_KERNEL_GAUSSIAN: return launchK32<FKTB_KERNEL_GAUSSIAN>(A, tiles, st);
    case FKTB_KERNEL_INVERSE_R: return launchK32<FKTB_KERNEL_INVERSE_R>(A, tiles, st);
    case FKTB_KERNEL_INVERSE_R2: return launchK32<FKTB_KERNEL_INVERSE_R2>(A, tiles, st);
    default: return false;
  }
}

}  // namespace fktb
