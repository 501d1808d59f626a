// Permutation gather/scatter around the MVM and K7 dense rows.
//
// K7 restates proj/src/transform.cpp:210-237 (denseMultiply): z_i =
// sum_j K(|x_i - x_j|) y_j with the r == 0 diagonal convention, for a list of
// rows (all rows for the full dense product). Grid = (row tiles, source
// splits); sources staged in shared memory like the near field.
#include "device_math.cuh"
#include "plan.hpp"

namespace fktb {
namespace {

// grid (positions / 256, right-hand sides): coalesced on the tree-order side;
// the original-order side is a permutation (a column stays L2-resident at the
// BASELINE sizes). 32-bit index math (no 64-bit division per element).
__global__ void gather_y(const double* __restrict__ y, const uint32_t* __restrict__ order, double* __restrict__ yp,
                         int n) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const size_t col = static_cast<size_t>(blockIdx.y) * n;
  yp[col + pos] = y[col + order[pos]];
}

__global__ void scatter_z(const double* __restrict__ zp, const uint32_t* __restrict__ order, double* __restrict__ z,
                          int n) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const size_t col = static_cast<size_t>(blockIdx.y) * n;
  z[col + order[pos]] = zp[col + pos];
}

constexpr int kDenseThreads = 128;
constexpr int kDenseRPT = 2;
constexpr int kDenseChunk = 512;

struct DenseArgs {
  int n, d, m;
  const double* x;  // row-major n x d
  const double* y;
  const int64_t* rows;
  double* z;
  int splitLen;
  FktbKernelDesc kd;
};

template <int KID>
__global__ void __launch_bounds__(kDenseThreads) dense_rows_kernel(const __grid_constant__ DenseArgs A) {
  extern __shared__ double smem[];
  double* sw = smem;
  double* sx = smem + kDenseChunk;  // [d][chunk]
  const int d = A.d;
  int row[kDenseRPT];
  double tx[kDenseRPT][FKTB_MAX_DIM];
  double acc[kDenseRPT];
#pragma unroll
  for (int i = 0; i < kDenseRPT; ++i) {
    const int q = blockIdx.x * (kDenseThreads * kDenseRPT) + threadIdx.x + i * kDenseThreads;
    row[i] = q < A.m ? q : -1;
    const long long src = row[i] >= 0 ? A.rows[q] : 0;
    for (int a = 0; a < d; ++a) tx[i][a] = A.x[src * d + a];
    acc[i] = 0.0;
  }
  const int s0 = blockIdx.y * A.splitLen;
  const int s1 = min(A.n, s0 + A.splitLen);
  for (int cs = s0; cs < s1; cs += kDenseChunk) {
    const int cn = min(kDenseChunk, s1 - cs);
    __syncthreads();
    for (int s = threadIdx.x; s < cn; s += kDenseThreads) {
      sw[s] = A.y[cs + s];
      for (int a = 0; a < d; ++a) sx[a * kDenseChunk + s] = A.x[static_cast<size_t>(cs + s) * d + a];
    }
    __syncthreads();
    for (int s = 0; s < cn; ++s) {
      const double w = sw[s];
#pragma unroll
      for (int i = 0; i < kDenseRPT; ++i) {
        double dist2 = 0.0;
        for (int a = 0; a < d; ++a) {
          const double t = tx[i][a] - sx[a * kDenseChunk + s];
          dist2 = fma(t, t, dist2);
        }
        double kv = kernel_value<KID>(A.kd, dist2);
        kv = dist2 == 0.0 ? A.kd.diag : kv;
        acc[i] = fma(kv, w, acc[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kDenseRPT; ++i)
    if (row[i] >= 0) atomicAdd(A.z + row[i], acc[i]);
}

template <int KID>
void launchDense(const DenseArgs& A, cudaStream_t st) {
  const int rowTiles = (A.m + kDenseThreads * kDenseRPT - 1) / (kDenseThreads * kDenseRPT);
  const int splits = (A.n + A.splitLen - 1) / A.splitLen;
  const size_t smem = static_cast<size_t>(kDenseChunk) * (A.d + 1) * sizeof(double);
  FKTB_CUDA(cudaFuncSetAttribute(dense_rows_kernel<KID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kDenseChunk * (FKTB_MAX_DIM + 1) * sizeof(double))));
  dense_rows_kernel<KID><<<dim3(rowTiles, splits), kDenseThreads, smem, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

}  // namespace

void launchGatherY(const DevicePlan& plan, const double* y, double* yp, int nrhs, cudaStream_t st) {
  gather_y<<<dim3((plan.n + 255) / 256, nrhs), 256, 0, st>>>(y, plan.tree->order.get(), yp, plan.n);
  FKTB_CUDA(cudaGetLastError());
}

void launchScatterZ(const DevicePlan& plan, const double* zp, double* z, int nrhs, cudaStream_t st) {
  scatter_z<<<dim3((plan.n + 255) / 256, nrhs), 256, 0, st>>>(zp, plan.tree->order.get(), z, plan.n);
  FKTB_CUDA(cudaGetLastError());
}

void denseRowsGpu(int n, int d, const double* dX, const FktbKernelDesc& kd, const double* dY, int m,
                  const int64_t* dRows, double* dZ, cudaStream_t st) {
  if (m <= 0) return;
  FKTB_CUDA(cudaMemsetAsync(dZ, 0, static_cast<size_t>(m) * sizeof(double), st));
  DenseArgs A{n, d, m, dX, dY, dRows, dZ, 0, kd};
  // Enough CTAs to fill 148 SMs several times over.
  const long long rowTiles = (m + kDenseThreads * kDenseRPT - 1) / (kDenseThreads * kDenseRPT);
  long long splits = std::max(1ll, (148ll * 8 + rowTiles - 1) / rowTiles);
  A.splitLen = static_cast<int>(std::max<long long>(kDenseChunk, (n + splits - 1) / splits));
  switch (kd.id) {
    case FKTB_KERNEL_EXPONENTIAL: return launchDense<FKTB_KERNEL_EXPONENTIAL>(A, st);
    case FKTB_KERNEL_MATERN12: return launchDense<FKTB_KERNEL_MATERN12>(A, st);
    case FKTB_KERNEL_MATERN32: return launchDense<FKTB_KERNEL_MATERN32>(A, st);
    case FKTB_KERNEL_CAUCHY: return launchDense<FKTB_KERNEL_CAUCHY>(A, st);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return launchDense<FKTB_KERNEL_RATIONAL_QUADRATIC>(A, st);
    case FKTB_KERNEL_GAUSSIAN: return launchDense<FKTB_KERNEL_GAUSSIAN>(A, st);
    case FKTB_KERNEL_INVERSE_R: return launchDense<FKTB_KERNEL_INVERSE_R>(A, st);
    case FKTB_KERNEL_INVERSE_R2: return launchDense<FKTB_KERNEL_INVERSE_R2>(A, st);
    case FKTB_KERNEL_INVERSE_R3: return launchDense<FKTB_KERNEL_INVERSE_R3>(A, st);
    case FKTB_KERNEL_EXP_OVER_R: return launchDense<FKTB_KERNEL_EXP_OVER_R>(A, st);
    case FKTB_KERNEL_R_EXP: return launchDense<FKTB_KERNEL_R_EXP>(A, st);
    case FKTB_KERNEL_COS_OVER_R: return launchDense<FKTB_KERNEL_COS_OVER_R>(A, st);
    case FKTB_KERNEL_EXP_NEG_INV_R: return launchDense<FKTB_KERNEL_EXP_NEG_INV_R>(A, st);
    case FKTB_KERNEL_EXP_NEG_INV_R2: return launchDense<FKTB_KERNEL_EXP_NEG_INV_R2>(A, st);
  }
  throw std::invalid_argument("dense: unknown kernel id");
}

}  // namespace fktb
