// Shared CUDA helpers: error checking, block reductions, warp primitives.
#ifndef FKTB_COMMON_CUH
#define FKTB_COMMON_CUH

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace fktb {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

inline void cudaCheck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

#define FKTB_CUDA(call) ::fktb::cudaCheck((call), #call)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide reductions (blockDim.x a multiple of 32, <= 1024). `scratch`
// holds >= 32 doubles. Result is broadcast to every thread.
template <int OP>  // 0 sum, 1 min, 2 max
__device__ __forceinline__ double block_reduce(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = OP == 0 ? warp_sum(v) : OP == 1 ? warp_min(v) : warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < nw ? scratch[lane] : (OP == 0 ? 0.0 : OP == 1 ? __longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double(0xfff0000000000000ll));
    w = OP == 0 ? warp_sum(w) : OP == 1 ? warp_min(w) : warp_max(w);
    if (lane == 0) scratch[0] = w;
  }
  __syncthreads();
  const double r = scratch[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_ll(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < nw ? scratch[lane] : 0;
    w = warp_sum_ll(w);
    if (lane == 0) scratch[0] = w;
  }
  __syncthreads();
  const long long r = scratch[0];
  __syncthreads();
  return r;
}

// Where the near / far kernels put the result of one (target, list entry): default, an FP64 atomic into z (tree order, n per right-hand side);
// deterministic plans (FktOptions::deterministic, det.cu), a plain store of
// the partial at its list entry, right-hand sides minor (coalesced: a tile's
// entries are consecutive), which a fixed-order per-target sum turns into z
// (bitwise reproducible).
struct ZOut {
  double* zp;        // n per RHS
  double* part;      // deterministic: partials [entry][rhs] (nullptr: atomics)
  long long stride;  // right-hand sides per entry (the pass)
  long long base;    // first entry of this list (near entries, then far entries)
  int n;
  __device__ __forceinline__ void add(int rhs, long long entry, int pos, double v) const {
    if (part)
      part[static_cast<size_t>(base + entry) * stride + rhs] = v;
    else
      atomicAdd(zp + static_cast<size_t>(rhs) * n + pos, v);
  }
};

}  // namespace fktb

#endif
