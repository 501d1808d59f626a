// FP64 / FP32 FMA-pipe peak microbenchmark (roofline denominator for the
// FP64-bound FKT kernels; MEASURED_PEAKS.json only carries HBM and bf16).
//
// FP64: the larger of two probes of the one FP64 datapath (DFMA and the FP64
// tensor core share it on B200, profiles/r01_probes.txt):
//   * DFMA: 148 SMs x 8 CTAs x 256 threads, 8 independent chains per thread;
//   * DMMA: mma.sync m8n8k4 f64, 8 independent accumulators per warp.
// Each probe first runs a warm-up launch (clocks up), then short bursts (~1-2
// ms: the kernel timed alone, before the board power limit pulls the clock
// down -- a 17 ms DFMA run measured 34.2 TF, the 1-2 ms bursts 36.8-37.0 on
// the same B200), two lengths x five repetitions; the best counts. FP32: the
// FFMA chains.
// Returns FLOP/s (FMA = 2 flops).
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/fkt_cuda.h"
#include "common.cuh"

namespace {

// x <- x * s + b with the multiplier s warp-uniform (a uniform-register
// operand) and b per thread: two register-pair operands per DFMA. With both
// s and b in vector registers (three register pairs per DFMA) the same loop
// measured 34.1 TF against 36.9 -- register-file operand bandwidth, not the
// FP64 pipe, then bounds it.
template <class T>
__global__ void fma_chain(T* out, int iters, T s) {
  T x[8];
  const T b = threadIdx.x * T(1e-3);
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = T(c) * T(0.5);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = fma(x[c], s, b);
  }
  T sum = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) sum += x[c];
  if (sum == T(-12345.678)) out[0] = sum;  // keep the chains alive
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void dmma_chain(double* out, int iters, double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
  const double x = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i], x, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -12345.678) out[0] = s;
}

// best FLOP/s of `launch(iters)` over run lengths and repetitions
template <class L>
double bestRate(L launch, double flopsPerIter, int baseIters) {
  cudaEvent_t e0, e1;
  FKTB_CUDA(cudaEventCreate(&e0));
  FKTB_CUDA(cudaEventCreate(&e1));
  launch(baseIters);  // warm-up: bring the clocks up
  double best = 0.0;
  for (int len : {1, 2}) {
    const int iters = baseIters * len;
    for (int rep = 0; rep < 5; ++rep) {
      FKTB_CUDA(cudaEventRecord(e0));
      launch(iters);
      FKTB_CUDA(cudaEventRecord(e1));
      FKTB_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      FKTB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::max(best, flopsPerIter * iters / (ms * 1e-3));
    }
  }
  FKTB_CUDA(cudaGetLastError());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

int smCount() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <class T>
double measureFma() {
  const int blocks = smCount() * 8, threads = 256;
  T* out = nullptr;
  FKTB_CUDA(cudaMalloc(&out, sizeof(T)));
  const double perIter = 2.0 * 8 * 16 * static_cast<double>(blocks) * threads;
  const double r = bestRate([&](int it) { fma_chain<T><<<blocks, threads>>>(out, it, T(1.0000001)); }, perIter,
                            sizeof(T) == 8 ? 250 : 500);
  cudaFree(out);
  return r;
}

double measureDmma() {
  const int blocks = smCount() * 8, threads = 256;
  double* out = nullptr;
  FKTB_CUDA(cudaMalloc(&out, sizeof(double)));
  const double warps = blocks * threads / 32.0;
  const double perIter = warps * 8 * (2.0 * 8 * 8 * 4);
  const double r = bestRate([&](int it) { dmma_chain<<<blocks, threads>>>(out, it, 1.0000001); }, perIter, 500);
  cudaFree(out);
  return r;
}

}  // namespace

extern "C" int fkt_fma_peak(int fp32, double* flops_per_s) {
  try {
    *flops_per_s = fp32 ? measureFma<float>() : std::max(measureFma<double>(), measureDmma());
    return FKT_OK;
  } catch (const std::exception&) {
    return FKT_ERR_CUDA;
  }
}

extern "C" int fkt_fp64_peaks(double* dfma_flops_per_s, double* dmma_flops_per_s) {
  try {
    *dfma_flops_per_s = measureFma<double>();
    *dmma_flops_per_s = measureDmma();
    return FKT_OK;
  } catch (const std::exception&) {
    return FKT_ERR_CUDA;
  }
}
