// Device CG and GP posterior mean (gp.cu; reference proj/include/fkt/gp.hpp).
#ifndef FKTB_GP_HPP
#define FKTB_GP_HPP

#include "plan.hpp"

namespace fktb {

// y -> K y + noise .* y on device vectors (reference NoisyOperator,
// gp.cpp:20-44): the kernel product through a plan (fast) or the dense K7
// rows (the reference's dense fallback).
struct DeviceNoisyOperator {
  int n = 0;
  DevicePlan* plan = nullptr;
  // dense path
  int d = 0;
  DeviceBuffer<double> dX;       // row-major n x d
  DeviceBuffer<int64_t> dRows;   // 0..n-1
  FktbKernelDesc kd{};
  DeviceBuffer<double> noise;
  double kernelDiagonal = 0.0;   // K(0) under the diagonal convention, 0 if singular
  void kernelProduct(const double* y, double* z, cudaStream_t st);
};

struct CgDiagnostics {
  int iterations = 0;
  double finalResidual = 0.0;
  bool converged = false;
  int restarts = 0;
};

double safeKernelDiagonal(const KernelSpec& k, bool hasDiagonal, double diagonal);

// cgSolve (gp.cpp:58-124) with x, rhs on the device. restartOnIncrease=true
// is the reference's rule (restart from the current iterate whenever |r|
// grows, gp.cpp:100-111); false runs textbook CG (additive option: CG
// residuals are not monotone, and the reference rule restarts on about every
// other iteration on the kernels of test_gp.cpp, which then stall).
CgDiagnostics cgSolveDevice(DeviceNoisyOperator& op, const double* dRhs, double tolerance, int maxIterations,
                            bool jacobi, double* dX, cudaStream_t st, bool restartOnIncrease = true);

struct GpDeviceOptions {
  PlanOptions fkt;
  double cgTolerance = 1e-10;
  int cgMaxIterations = 1000;
  bool jacobi = false;
  bool dense = false;
  bool hasPriorMean = false;
  double priorMean = 0.0;
  bool restartOnIncrease = true;
};

// gpPosteriorMean (gp.cpp:126-177); host buffers in and out.
CgDiagnostics gpPosteriorMeanGpu(int nTrain, int d, const double* trainX, const double* y, const double* noise,
                                 const KernelSpec& kernel, int nTest, const double* testX, const GpDeviceOptions& o,
                                 double* mean);

// Dense operator setup shared by the C-ABI entry points.
void setupDenseOperator(DeviceNoisyOperator& op, int n, int d, const double* hostX, const KernelSpec& k,
                        bool hasDiagonal, double diagonal, cudaStream_t st);

}  // namespace fktb

#endif
