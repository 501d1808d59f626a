// Shared pieces of the FP64 near-field kernels (near.cu, nearsym.cu):
// canonical kernel bodies on pre-scaled coordinates and the scale factors.
#ifndef FKTB_NEAR_COMMON_CUH
#define FKTB_NEAR_COMMON_CUH

#include <cmath>

#include "fastmath.cuh"
#include "fkt_device_types.h"

namespace fktb {

template <int KID>
struct FastKernel {
  static constexpr bool supported =
      KID == FKTB_KERNEL_MATERN32 || KID == FKTB_KERNEL_MATERN12 || KID == FKTB_KERNEL_EXPONENTIAL ||
      KID == FKTB_KERNEL_CAUCHY || KID == FKTB_KERNEL_RATIONAL_QUADRATIC || KID == FKTB_KERNEL_GAUSSIAN ||
      KID == FKTB_KERNEL_INVERSE_R || KID == FKTB_KERNEL_INVERSE_R2;
  static constexpr bool needsTable =
      KID == FKTB_KERNEL_MATERN32 || KID == FKTB_KERNEL_MATERN12 || KID == FKTB_KERNEL_EXPONENTIAL ||
      KID == FKTB_KERNEL_GAUSSIAN;
  // canonical K at scaled squared distance q (> 0 unless the select handles 0)
  template <int REP>
  __device__ static __forceinline__ double eval(double q, const double* tab) {
    if constexpr (KID == FKTB_KERNEL_MATERN32) {
      const double u = sqrt_nr(q);
      const double e = exp_neg<REP, kNearExpBits>(u, tab);
      return fma(u, e, e);
    } else if constexpr (KID == FKTB_KERNEL_MATERN12 || KID == FKTB_KERNEL_EXPONENTIAL) {
      return exp_neg<REP, kNearExpBits>(sqrt_nr(q), tab);
    } else if constexpr (KID == FKTB_KERNEL_CAUCHY) {
      return rcp_nr(1.0 + q);
    } else if constexpr (KID == FKTB_KERNEL_RATIONAL_QUADRATIC) {
      return rsqrt_nr(1.0 + q);
    } else if constexpr (KID == FKTB_KERNEL_GAUSSIAN) {
      return exp_neg<REP, kNearExpBits>(q, tab);
    } else if constexpr (KID == FKTB_KERNEL_INVERSE_R) {
      return rsqrt_nr(q);
    } else {
      return rcp_nr(q);
    }
  }
};

// (scale for coordinates, prefactor for weights)
inline void fastScales(const FktbKernelDesc& k, double& sc, double& wf) {
  sc = 1.0;
  wf = 1.0;
  switch (k.id) {
    case FKTB_KERNEL_MATERN32: sc = k.a; wf = k.s2; break;
    case FKTB_KERNEL_MATERN12: sc = 1.0 / k.rho; wf = k.s2; break;
    case FKTB_KERNEL_CAUCHY:
    case FKTB_KERNEL_RATIONAL_QUADRATIC: sc = std::sqrt(k.is2); break;
    default: break;
  }
}

}  // namespace fktb

#endif
