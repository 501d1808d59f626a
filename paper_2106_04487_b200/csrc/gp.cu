// Device-resident conjugate gradients and the GP posterior mean
// (reference proj/src/gp.cpp:20-177, proj/include/fkt/gp.hpp).
//
// The reference's CG keeps every vector on the host and calls the FKT plan's
// multiply (H2D y, MVM, D2H z) once per iteration. Here the whole solve stays
// in HBM: x, r, z, p, Ap live on the device; each iteration is one device MVM
// (a replayed CUDA graph) plus five small vector kernels, and the host only
// reads two scalars (p.Ap and |r|^2) per iteration to take the reference's
// control decisions (break on p.Ap <= 0, monotonicity restart, tolerance).
//
// Dot products are deterministic: a fixed grid writes per-block partials in a
// grid-stride order and a single block reduces them in a fixed tree order;
// kernels that need a finished scalar (alpha, beta) read it from device
// memory, so no host round trip sits between the MVM and the updates.
#include <cmath>
#include <numeric>

#include "common.cuh"
#include "plan.hpp"
#include "gp.hpp"

namespace fktb {
namespace {

constexpr int kVecThreads = 256;
constexpr int kVecBlocks = 148 * 4;

enum Slot { kPap = 0, kRes2 = 1, kRz = 2, kRzNew = 3, kB2 = 4, kSlots = 8 };

__device__ __forceinline__ void block_partial(double v, double* partials) {
  __shared__ double red[kVecThreads / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < kVecThreads / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
  }
}

#define GRID_STRIDE(i, n) \
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); i += static_cast<long long>(gridDim.x) * blockDim.x)

__global__ void reduce_kernel(const double* partials, int count, double* scal, int slot) {
  __shared__ double red[kVecThreads];
  double t = 0.0;
  for (int i = threadIdx.x; i < count; i += kVecThreads) t += partials[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int s = kVecThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) scal[slot] = red[0];
}

// sum v^2
__global__ void sq_kernel(const double* v, long long n, double* partials) {
  double s = 0.0;
  GRID_STRIDE(i, n) s = fma(v[i], v[i], s);
  block_partial(s, partials);
}

// ap += noise .* p ; partial p . ap
__global__ void noise_dot_kernel(double* ap, const double* noise, const double* p, long long n, double* partials) {
  double s = 0.0;
  GRID_STRIDE(i, n) {
    const double a = fma(noise[i], p[i], ap[i]);
    ap[i] = a;
    s = fma(p[i], a, s);
  }
  block_partial(s, partials);
}

// if p.Ap > 0: alpha = rz / pAp; x += alpha p; r -= alpha Ap ; partial r.r
__global__ void update_xr_kernel(double* x, double* r, const double* p, const double* ap, const double* scal, long long n,
                                 double* partials) {
  const double pap = scal[kPap];
  double s = 0.0;
  if (pap > 0.0) {
    const double alpha = scal[kRz] / pap;
    GRID_STRIDE(i, n) {
      x[i] = fma(alpha, p[i], x[i]);
      const double ri = fma(-alpha, ap[i], r[i]);
      r[i] = ri;
      s = fma(ri, ri, s);
    }
  }
  block_partial(s, partials);
}

// z = pre .* r (pre == nullptr: z = r) ; partial r . z
__global__ void precond_dot_kernel(double* z, const double* r, const double* pre, long long n, double* partials) {
  double s = 0.0;
  GRID_STRIDE(i, n) {
    const double zi = pre ? pre[i] * r[i] : r[i];
    z[i] = zi;
    s = fma(r[i], zi, s);
  }
  block_partial(s, partials);
}

// p = z + (rzNew / rz) p
__global__ void update_p_kernel(double* p, const double* z, const double* scal, long long n) {
  const double beta = scal[kRzNew] / scal[kRz];
  GRID_STRIDE(i, n) p[i] = fma(beta, p[i], z[i]);
}

// r = rhs - (Kx + noise .* x)
__global__ void residual_kernel(double* r, const double* rhs, const double* kx, const double* noise, const double* x,
                                long long n) {
  GRID_STRIDE(i, n) r[i] = rhs[i] - fma(noise[i], x[i], kx[i]);
}

// Jacobi: pre = 1 / (K(0) + noise) where positive, else 1 (gp.cpp:74-81)
__global__ void jacobi_kernel(double* pre, const double* noise, double k0, long long n) {
  GRID_STRIDE(i, n) {
    const double d = k0 + noise[i];
    pre[i] = d > 0.0 ? 1.0 / d : 1.0;
  }
}

}  // namespace

double safeKernelDiagonal(const KernelSpec& k, bool hasDiagonal, double diagonal) {
  // gp.cpp:10-16: kernel(0, diagonal), 0 when singular without a convention
  if (hasDiagonal) return diagonal;
  return k.valueAtZero ? *k.valueAtZero : 0.0;
}

void DeviceNoisyOperator::kernelProduct(const double* y, double* z, cudaStream_t st) {
  if (plan) {
    multiplyDevice(*plan, y, z, 1, st);
  } else {
    denseRowsGpu(n, d, dX.get(), kd, y, n, dRows.get(), z, st);
  }
}

CgDiagnostics cgSolveDevice(DeviceNoisyOperator& op, const double* dRhs, double tolerance, int maxIterations,
                            bool jacobi, double* dX, cudaStream_t st, bool restartOnIncrease) {
  if (!(tolerance > 0.0)) throw std::invalid_argument("cgSolve requires a positive tolerance");
  const long long n = op.n;
  CgDiagnostics out;
  DeviceBuffer<double> r(n), z(n), p(n), ap(n), pre(jacobi ? n : 0), part(kVecBlocks), scal(kSlots);
  double hs[kSlots];
  auto reduce = [&](int slot) {
    reduce_kernel<<<1, kVecThreads, 0, st>>>(part.get(), kVecBlocks, scal.get(), slot);
    FKTB_CUDA(cudaGetLastError());
  };
  auto fetch = [&]() {
    FKTB_CUDA(cudaMemcpyAsync(hs, scal.get(), sizeof(hs), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaStreamSynchronize(st));
  };
  FKTB_CUDA(cudaMemsetAsync(dX, 0, n * sizeof(double), st));
  FKTB_CUDA(cudaMemsetAsync(scal.get(), 0, scal.bytes(), st));
  sq_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(dRhs, n, part.get());
  reduce(kB2);
  fetch();
  const double bNorm = std::sqrt(hs[kB2]);
  if (bNorm == 0.0) {
    out.converged = true;
    return out;
  }
  const double* preP = nullptr;
  if (jacobi) {
    jacobi_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(pre.get(), op.noise.get(), op.kernelDiagonal, n);
    preP = pre.get();
  }
  // r = b; z = M r; p = z; rz = r.z; |r|
  FKTB_CUDA(cudaMemcpyAsync(r.get(), dRhs, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  precond_dot_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(z.get(), r.get(), preP, n, part.get());
  reduce(kRz);
  FKTB_CUDA(cudaMemcpyAsync(p.get(), z.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  double resNorm = bNorm;  // r == b
  int iter = 0;
  while (iter < maxIterations && resNorm / bNorm > tolerance) {
    ++iter;
    op.kernelProduct(p.get(), ap.get(), st);
    noise_dot_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(ap.get(), op.noise.get(), p.get(), n, part.get());
    reduce(kPap);
    update_xr_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(dX, r.get(), p.get(), ap.get(), scal.get(), n, part.get());
    reduce(kRes2);
    fetch();
    if (hs[kPap] <= 0.0) break;  // loss of positive definiteness under roundoff (gp.cpp:94)
    const double newRes = std::sqrt(hs[kRes2]);
    if (restartOnIncrease && newRes > resNorm) {
      // Monotonicity restart from the current iterate (gp.cpp:100-111)
      op.kernelProduct(dX, ap.get(), st);
      residual_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(r.get(), dRhs, ap.get(), op.noise.get(), dX, n);
      precond_dot_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(z.get(), r.get(), preP, n, part.get());
      reduce(kRz);
      FKTB_CUDA(cudaMemcpyAsync(p.get(), z.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      sq_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(r.get(), n, part.get());
      reduce(kRes2);
      fetch();
      resNorm = std::sqrt(hs[kRes2]);
      ++out.restarts;
      continue;
    }
    resNorm = newRes;
    precond_dot_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(z.get(), r.get(), preP, n, part.get());
    reduce(kRzNew);
    update_p_kernel<<<kVecBlocks, kVecThreads, 0, st>>>(p.get(), z.get(), scal.get(), n);
    FKTB_CUDA(cudaMemcpyAsync(scal.get() + kRz, scal.get() + kRzNew, sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  FKTB_CUDA(cudaGetLastError());
  FKTB_CUDA(cudaStreamSynchronize(st));
  out.iterations = iter;
  out.finalResidual = resNorm / bNorm;
  out.converged = resNorm / bNorm <= tolerance;
  return out;
}

void setupDenseOperator(DeviceNoisyOperator& op, int n, int d, const double* hostX, const KernelSpec& k,
                        bool hasDiagonal, double diagonal, cudaStream_t st) {
  if (d < 1 || d > FKTB_MAX_DIM) throw std::invalid_argument("unsupported on the GPU path: dense products need 1 <= d <= 16");
  fillKernelDesc(k, op.kd);
  if (hasDiagonal)
    op.kd.diag = diagonal;
  else if (!k.valueAtZero)
    throw std::domain_error("kernel '" + k.name + "' is singular at r = 0 and no diagonal convention is set");
  op.plan = nullptr;
  op.n = n;
  op.d = d;
  op.dX.resize(static_cast<size_t>(n) * d);
  FKTB_CUDA(cudaMemcpyAsync(op.dX.get(), hostX, op.dX.bytes(), cudaMemcpyHostToDevice, st));
  std::vector<int64_t> rows(static_cast<size_t>(n));
  std::iota(rows.begin(), rows.end(), 0);
  op.dRows.resize(static_cast<size_t>(n));
  FKTB_CUDA(cudaMemcpyAsync(op.dRows.get(), rows.data(), op.dRows.bytes(), cudaMemcpyHostToDevice, st));
  FKTB_CUDA(cudaStreamSynchronize(st));  // rows is a host temporary
}

CgDiagnostics gpPosteriorMeanGpu(int nTrain, int d, const double* trainX, const double* y, const double* noise,
                                 const KernelSpec& kernel, int nTest, const double* testX, const GpDeviceOptions& o,
                                 double* mean) {
  // prior mean: given, else the mean of the targets (gp.cpp:133-135)
  const double mu = o.hasPriorMean ? o.priorMean : std::accumulate(y, y + nTrain, 0.0) / static_cast<double>(nTrain);
  std::vector<double> resid(static_cast<size_t>(nTrain));
  for (int i = 0; i < nTrain; ++i) resid[static_cast<size_t>(i)] = y[i] - mu;
  cudaStream_t st;
  FKTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamSynchronize(s), cudaStreamDestroy(s); }
  } guard{st};
  DeviceNoisyOperator op;
  std::unique_ptr<DevicePlan, void (*)(DevicePlan*)> trainPlan(nullptr, destroyPlan);
  if (o.dense) {
    setupDenseOperator(op, nTrain, d, trainX, kernel, o.fkt.hasDiagonal, o.fkt.diagonal, st);
  } else {
    trainPlan.reset(createPlan(nTrain, d, trainX, kernel, o.fkt).release());
    op.plan = trainPlan.get();
    op.n = nTrain;
  }
  op.kernelDiagonal = safeKernelDiagonal(kernel, o.fkt.hasDiagonal, o.fkt.diagonal);
  op.noise.resize(static_cast<size_t>(nTrain));
  FKTB_CUDA(cudaMemcpyAsync(op.noise.get(), noise, op.noise.bytes(), cudaMemcpyHostToDevice, st));
  DeviceBuffer<double> dResid(static_cast<size_t>(nTrain));
  FKTB_CUDA(cudaMemcpyAsync(dResid.get(), resid.data(), dResid.bytes(), cudaMemcpyHostToDevice, st));
  const int nJ = nTrain + nTest;
  DeviceBuffer<double> padded(static_cast<size_t>(nJ)), cross(static_cast<size_t>(nJ));
  FKTB_CUDA(cudaMemsetAsync(padded.get(), 0, padded.bytes(), st));
  // the solution lands directly in the train block of the zero-padded source vector
  const CgDiagnostics diag =
      cgSolveDevice(op, dResid.get(), o.cgTolerance, o.cgMaxIterations, o.jacobi, padded.get(), st, o.restartOnIncrease);
  trainPlan.reset();
  // Cross product k(X*, X) v on the concatenated cloud (gp.cpp:153-170)
  std::vector<double> joint(static_cast<size_t>(nJ) * d);
  std::copy(trainX, trainX + static_cast<size_t>(nTrain) * d, joint.begin());
  std::copy(testX, testX + static_cast<size_t>(nTest) * d, joint.begin() + static_cast<size_t>(nTrain) * d);
  double* testPart = nullptr;
  if (o.dense) {
    // only the test rows of the dense product are read; evaluate just those
    DeviceNoisyOperator jop;
    setupDenseOperator(jop, nJ, d, joint.data(), kernel, o.fkt.hasDiagonal, o.fkt.diagonal, st);
    denseRowsGpu(nJ, d, jop.dX.get(), jop.kd, padded.get(), nTest, jop.dRows.get() + nTrain, cross.get(), st);
    testPart = cross.get();
    FKTB_CUDA(cudaMemcpyAsync(mean, testPart, static_cast<size_t>(nTest) * sizeof(double), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaStreamSynchronize(st));
  } else {
    PlanOptions jo = o.fkt;
    jo.eagerOperators = false;  // single multiply (gp.cpp:165)
    std::unique_ptr<DevicePlan, void (*)(DevicePlan*)> jointPlan(createPlan(nJ, d, joint.data(), kernel, jo).release(),
                                                                 destroyPlan);
    jointPlan->useGraphs = false;  // one multiply: no capture
    multiplyDevice(*jointPlan, padded.get(), cross.get(), 1, st);
    testPart = cross.get() + nTrain;
    FKTB_CUDA(cudaMemcpyAsync(mean, testPart, static_cast<size_t>(nTest) * sizeof(double), cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaStreamSynchronize(st));
  }
  for (int i = 0; i < nTest; ++i) mean[i] += mu;
  return diag;
}

}  // namespace fktb
