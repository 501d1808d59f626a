// FP64 / FP32 FMA-pipe peak microbenchmark (roofline denominator for the
// FP64-bound FKT kernels; MEASURED_PEAKS.json only carries HBM and bf16).
// Grid = 148 SMs x 8 CTAs x 256 threads, 8 independent FMA chains per thread,
// timed with CUDA events; returns FLOP/s (FMA = 2 flops).
#include <cuda_runtime.h>

#include "../../include/fkt_cuda.h"
#include "common.cuh"

namespace {

template <class T>
__global__ void fma_chain(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x * T(1e-3), x1 = x0 + T(1), x2 = x0 + T(2), x3 = x0 + T(3);
  T x4 = x0 + T(4), x5 = x0 + T(5), x6 = x0 + T(6), x7 = x0 + T(7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b);
      x1 = fma(x1, a, b);
      x2 = fma(x2, a, b);
      x3 = fma(x3, a, b);
      x4 = fma(x4, a, b);
      x5 = fma(x5, a, b);
      x6 = fma(x6, a, b);
      x7 = fma(x7, a, b);
    }
  }
  const T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == T(-12345.678)) out[0] = s;  // keep the chains alive
}

template <class T>
double measure(int iters) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  T* out = nullptr;
  FKTB_CUDA(cudaMalloc(&out, sizeof(T)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_chain<T><<<blocks, threads>>>(out, iters / 10, T(0.999999), T(1e-7));  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_chain<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  FKTB_CUDA(cudaGetLastError());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
  return flops / (best * 1e-3);
}

}  // namespace

extern "C" int fkt_fma_peak(int fp32, double* flops_per_s) {
  try {
    *flops_per_s = fp32 ? measure<float>(4000) : measure<double>(2000);
    return FKT_OK;
  } catch (const std::exception&) {
    return FKT_ERR_CUDA;
  }
}
