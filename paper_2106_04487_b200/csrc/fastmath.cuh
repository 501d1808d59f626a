// FP64 elementary functions for the near-field pair loop (sm_100a).
//
// The pair loop is bound by FP64-pipe issue, so these trade the last bits of
// libm's correctly rounded results for fewer instructions while keeping a
// relative error <= ~5e-14 per evaluation (z is gated at rel-L2 1e-10):
//   * exp_neg(u) = e^-u, u >= 0: 2^(j/2^BITS) table in shared memory,
//     one-constant range reduction, Taylor polynomial (BITS = 6: 64 entries,
//     degree 4, 8 FP64 ops -- the far kernels; BITS = 9: 512 entries, degree
//     3, 7 FP64 ops -- the near field, measured -6.5% K3 time at cfg2),
//     exponent added in the integer pipe.
//   * rsqrt_nr / sqrt_nr: MUFU rsqrt.approx.f64 + one Newton step. 4 FP64 ops.
//   * rcp_nr: MUFU rcp.approx.f64 + one Newton step. 2 FP64 ops.
#ifndef FKTB_FASTMATH_CUH
#define FKTB_FASTMATH_CUH

#include <cstdint>

namespace fktb {

constexpr int kExpTable = 64;
// Shared-memory copy: entry j replicated for 16 bank pairs,
// tab[j * kExpRep + c]; lane L reads column L % 16 so a warp's 64-bit lookups
// never conflict (ncu showed 3.9-way conflicts with a single copy).
constexpr int kExpRep = 16;
// Added to every squared pair distance: keeps rsqrt finite at r == 0 and is
// below one ulp of any squared distance >= 1e-284.
constexpr double kQBias = 1e-300;

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// 1/sqrt(x), x > 0.
__device__ __forceinline__ double rsqrt_nr(double x) {
  const double y0 = rsqrt_approx(x);
  const double h = x * y0;
  const double e = fma(-h, y0, 1.0);
  return fma(0.5 * y0, e, y0);
}

// sqrt(x) for x > 0 (callers bias squared distances by kQBias so x == 0
// never reaches the approximation's infinity).
__device__ __forceinline__ double sqrt_nr(double x) {
  const double y0 = rsqrt_approx(x);
  const double h = x * y0;
  const double e = fma(-h, y0, 1.0);
  return fma(0.5 * h, e, h);
}

// 1/x, x normal: two Newton steps (the MUFU seed has ~2^-23 relative error;
// one step leaves ~1e-14, two reach rounding level, which the reference's
// single-leaf exactness test (1e-13 vs dense) needs).
__device__ __forceinline__ double rcp_nr(double x) {
  const double y0 = rcp_approx(x);
  const double e0 = fma(-x, y0, 1.0);
  const double y1 = fma(y0, e0, y0);
  const double e1 = fma(-x, y1, 1.0);
  return fma(y1, e1, y1);
}

// Near-field table: 2^NEAR_EXP_BITS entries (9 -> 512 entries, 4 KB of shared
// memory, |f| <= ln2/1024 so a degree-3 polynomial suffices: one FP64 op per
// pair fewer than the 64-entry / degree-4 table; cfg2 K3 14.72 -> 13.76 ms).
#ifndef FKTB_NEAR_EXP_BITS
#define FKTB_NEAR_EXP_BITS 9
#endif
constexpr int kNearExpBits = FKTB_NEAR_EXP_BITS;
constexpr int kNearExpTable = 1 << kNearExpBits;

// e^-u for u >= 0 (underflows to ~0 past u = 708). tab: the lane's column of
// the replicated 2^(j/2^BITS) table (tab[j * REP] = 2^(j/2^BITS)).
template <int REP = kExpRep, int BITS = 6>
__device__ __forceinline__ double exp_neg(double u, const double* __restrict__ tab) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  constexpr double kInvStep = 1.4426950408889634 * (1 << BITS);  // 2^BITS / ln 2 (exact power-of-two scaling)
  // ln2/2^BITS rounded to double: a one-constant reduction errs by |k| * 2^-60,
  // i.e. <= u * 1e-16 relative in e^-u (a two-constant Cody-Waite step would
  // cost one more FP64 op per pair for accuracy the 1e-10 gate does not need).
  constexpr double kStep = 0.6931471805599453 / (1 << BITS);
  // clamp u <= ~708 on the high word (integer pipe): e^-708 ~ 3e-308, and
  // keeps the exponent arithmetic below in the normal range
  u = __hiloint2double(min(__double2hiint(u), 0x40862000), __double2loint(u));
  const double t = fma(-u, kInvStep, kMagic);
  const int k = __double2loint(t);  // round(-u * 2^BITS / ln2), <= 0
  const double kd = t - kMagic;
  const double f = fma(kd, -kStep, -u);
  double p;
  if constexpr (BITS >= 9) {  // |f| <= 6.8e-4: degree 3, truncation f^4/24 < 9e-15
    p = fma(f, 1.0 / 6.0, 0.5);
  } else {  // |f| <= 5.4e-3: degree 4, truncation f^5/120 < 4e-14
    p = fma(f, 1.0 / 24.0, 1.0 / 6.0);
    p = fma(f, p, 0.5);
  }
  p = fma(f, p, 1.0);
  p = fma(f, p, 1.0);
  const double tj = tab[(k & ((1 << BITS) - 1)) * REP];
  const int e = k >> BITS;  // arithmetic shift: floor(k / 2^BITS)
  const double scaled = __hiloint2double(__double2hiint(tj) + (e << 20), __double2loint(tj));
  return scaled * p;
}

}  // namespace fktb

#endif

#ifndef FKTB_FASTMATH_FILL
#define FKTB_FASTMATH_FILL
namespace fktb {
// Fill the replicated shared table from the 64-entry device table.
__device__ __forceinline__ void fill_exp_table(double* tab, const double* src) {
  for (int i = threadIdx.x; i < kExpTable * kExpRep; i += blockDim.x) tab[i] = src[i / kExpRep];
}
}  // namespace fktb
#endif
