// Shared pieces of the FP64 near-field kernels (near.cu):
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
  // Gram-form pair distances (near.cu): q = |t|^2 + |s|^2 - 2 t.s on
  // leaf-centred coordinates, with `gramOffset` folded into |s|^2 (the 1 + r^2
  // of the Cauchy family). Only for kernels whose K is smooth in q (bounded
  // dK/dq, so the q rounding of eps * (|t|^2 + |s|^2) stays an absolute error
  // of the same size) and that need no exact r == 0 detection.
  // (Not the exponential / Matern-1/2 kernels: e^-sqrt(q) has an unbounded
  // dK/dq at 0, so a 1e-15 error in q becomes ~3e-8 in K.)
  static constexpr bool gram = KID == FKTB_KERNEL_MATERN32 || KID == FKTB_KERNEL_CAUCHY ||
                               KID == FKTB_KERNEL_RATIONAL_QUADRATIC || KID == FKTB_KERNEL_GAUSSIAN;
  // The Gaussian's offset 1 keeps its exp argument q + 1 >= ~1 (q may round
  // below 0) and the factor e rides on the weights: e^-q = e * e^-(q + 1).
  static constexpr double gramOffset =
      KID == FKTB_KERNEL_CAUCHY || KID == FKTB_KERNEL_RATIONAL_QUADRATIC || KID == FKTB_KERNEL_GAUSSIAN ? 1.0 : 0.0;
  static constexpr double gramWeight = KID == FKTB_KERNEL_GAUSSIAN ? 2.718281828459045 : 1.0;
  // Gaussian, factored Gram form (near.cu near_tile): e^-q = e^-|t|^2 *
  // (e^(B - |s|^2) w) * e^-(B - 2 t.s), B the tile bound: d FMAs per pair and
  // no add (the |t|^2 factor is applied once per target).
  static constexpr bool gramFactored = KID == FKTB_KERNEL_GAUSSIAN;
  // Matern-3/2 takes sqrt(q): its Gram q gets an additive bias (near.cu).
  static constexpr bool gramBiased = KID == FKTB_KERNEL_MATERN32;

  // Matern-3/2's Gram rows carry TWICE the squared distance (sqrt_nr_half).
  static constexpr double gramScale = KID == FKTB_KERNEL_MATERN32 ? 2.0 : 1.0;

  template <int REP, bool CLAMP_LO = true, bool CLAMP_HI = true>
  __device__ static __forceinline__ double expn(double u, const double* tab, int colBytes) {
    return exp_neg_fi<REP, kNearExpBits, CLAMP_LO, CLAMP_HI>(u, tab, colBytes);
  }

  // canonical K at scaled squared distance q (> 0 unless the select handles
  // 0); GRAM: q already carries gramOffset and gramScale. tab: the
  // REP-replicated, pre-compensated exp table (exp_neg_fi), colBytes: 8 *
  // this lane's column.
  template <int REP, bool GRAM = false>
  __device__ static __forceinline__ double eval(double q, const double* tab, int colBytes = 0) {
    // Gram q may round slightly below 0: Matern's sources carry a bias that
    // covers the rounding (near.cu gramBias), the other Gram kernels take 1 + q. The Gram
    // bound keeps sqrt(q) and 1 + q far below the exp clamp: no clamps here.
    if constexpr (KID == FKTB_KERNEL_MATERN32) {
      double u = GRAM ? sqrt_nr_half(q) : sqrt_nr(q);  // Gram q = 2 r^2
      if constexpr (!GRAM) u = clamp_exp_arg(u);  // in place: the (1 + u) factor uses the same u
      const double e = expn<REP, !GRAM, false>(u, tab, colBytes);
      return fma(u, e, e);
    } else if constexpr (KID == FKTB_KERNEL_MATERN12 || KID == FKTB_KERNEL_EXPONENTIAL) {
      return expn<REP, !GRAM, true>(sqrt_nr(q), tab, colBytes);
    } else if constexpr (KID == FKTB_KERNEL_CAUCHY) {
      return rcp_nr(GRAM ? q : 1.0 + q);
    } else if constexpr (KID == FKTB_KERNEL_RATIONAL_QUADRATIC) {
      return rsqrt_nr(GRAM ? q : 1.0 + q);
    } else if constexpr (KID == FKTB_KERNEL_GAUSSIAN) {
      return expn<REP, !GRAM, !GRAM>(q, tab, colBytes);
    } else if constexpr (KID == FKTB_KERNEL_INVERSE_R) {
      return rsqrt_nr_half(q);  // q = r^2 / 2: fastScales scales by 1/sqrt(2)
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
    case FKTB_KERNEL_INVERSE_R: sc = std::sqrt(0.5); break;  // eval takes r^2 / 2 (rsqrt_nr_half)
    default: break;
  }
}

}  // namespace fktb

#endif
