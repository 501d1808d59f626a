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
constexpr int kQBiasHi = 0x01a56e1f;  // high word of kQBias

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

// 1/sqrt(2 x) for x > 0: callers pass HALF the squared distance, so the
// Newton step's factor 1/2 rides on the argument (3 FP64 ops, not 4). The
// seed is MUFU rsqrt of 2x, formed on the high word (exponent + 1).
__device__ __forceinline__ double rsqrt_nr_half(double x) {
  const double y0 = rsqrt_approx(__hiloint2double(__double2hiint(x) + 0x00100000, 0));
  const double h = x * y0;
  const double e = fma(-h, y0, 0.5);  // (1 - 2 x y0^2) / 2
  return fma(y0, e, y0);
}

// sqrt(x / 2) for x > 0: callers pass TWICE the squared distance (Gram rows
// scaled by 2), so the Newton step's factor 1/2 rides on the argument and the
// step costs 3 FP64 ops (DMUL + 2 DFMA) instead of 4. The seed is MUFU rsqrt
// of 2x (exponent + 1 on the high word, integer pipe): y0 ~ 1/sqrt(2x),
// h = x y0 ~ sqrt(x/2), e = 1/2 - h y0 = -(delta + delta^2/2) for the seed
// error delta, and h (1 + e) has error O(delta^2).
__device__ __forceinline__ double sqrt_nr_half(double x) {
  const double y0 = rsqrt_approx(__hiloint2double(__double2hiint(x) + 0x00100000, 0));
  const double h = x * y0;
  const double e = fma(-h, y0, 0.5);
  return fma(h, e, h);
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

// Near-field table: 2^NEAR_EXP_BITS entries. 10 -> 1024 entries (8 KB per
// one-warp CTA), degree-2 remainder (exp_neg_fi below). Round-1 alternative:
// 64 entries replicated for the 16 bank pairs (conflict-free lookups) with
// degree 4 was 6% slower than 512 entries with degree 3.
#ifndef FKTB_NEAR_EXP_BITS
#define FKTB_NEAR_EXP_BITS 10
#endif
constexpr int kNearExpBits = FKTB_NEAR_EXP_BITS;
constexpr int kNearExpTable = 1 << kNearExpBits;
constexpr int kNearExpRep = kNearExpBits <= 7 ? kExpRep : 1;

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

// Near-field e^-u (exp_neg_fi): e^-u = 2^(k/2^BITS) e^f with
// k = round(-u 2^BITS / ln2) taken from the low word of one magic-number DFMA,
// f = -k ln2/2^BITS - u by one more DFMA (|f| <= half a table step), a
// degree-2 remainder from BITS = 10 on (1024-entry table: |f| <= 3.4e-4,
// truncation f^3/6 <= 6.5e-12 relative; measured z error vs the reference FKT
// 1.7e-12 at cfg2, gate 1e-10), and the exponent of k folded into the table
// entry's high word by one integer shift-add (pre-compensated table).
// Round-2 B200 measurements behind this form (cfg2 near field, 11.55 ms with
// a 512-entry table, degree 3 and an FP32-pipe index = 15 FP64 + 11 other
// instructions per pair): degree 2 at 1024 entries 11.21 ms; the index by DFMA
// instead of LEA + FFMA + MOV 11.51 ms; both 10.78 ms. The pair loop runs at
// ~2 issue cycles per FP64 instruction plus ~1 per other instruction
// (register-file operand bandwidth, scripts/probes/rf_probe.cu), so an FP64
// op that replaces three integer/FP32 ones is a gain.
//   CLAMP_HI: clamp u <= ~708.3 here (else the caller did, see clamp_exp_arg).
//   CLAMP_LO: kept for the callers' intent (u below 2^-127 or slightly
//     negative gives k = 0 and f = -u in this form without any clamp).
__device__ __forceinline__ double clamp_exp_arg(double u) {
  return __hiloint2double(min(__double2hiint(u), 0x40862000), __double2loint(u));
}

// Table lookup of entry (k mod 2^BITS) in the REP-replicated shared table at
// `tab` (entry j, column c at tab[j * REP + c]); colBytes = 8 * the lane's
// column. One shift and one LOP3 (and | or) give the byte offset.
template <int REP, int BITS>
__device__ __forceinline__ double exp_table_at(const double* __restrict__ tab, int k, int colBytes) {
  static_assert((REP & (REP - 1)) == 0, "REP must be a power of two");
  constexpr int kLog = REP == 1 ? 0 : REP == 2 ? 1 : REP == 4 ? 2 : REP == 8 ? 3 : 4;
  static_assert((1 << kLog) == REP, "REP <= 16");
  const unsigned off = ((static_cast<unsigned>(k) << (3 + kLog)) & (((1u << BITS) - 1u) << (3 + kLog))) |
                       static_cast<unsigned>(colBytes);
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab) + off);
}

#ifndef FKTB_EXP_DEG2_BITS
#define FKTB_EXP_DEG2_BITS 10  // table bits from which the degree-2 polynomial is used
#endif
// tab: the PRE-COMPENSATED table (see the exponent step below).
template <int REP = 1, int BITS = 9, bool CLAMP_LO = true, bool CLAMP_HI = true>
__device__ __forceinline__ double exp_neg_fi(double u, const double* __restrict__ tab, int colBytes) {
  static_assert(BITS >= 6, "degree-4 polynomial needs |f| <= ln2/2^7");
  constexpr double kInvStep = 1.4426950408889634 * (1 << BITS);
  constexpr double kStep = 0.6931471805599453 / (1 << BITS);
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  if constexpr (CLAMP_HI) u = clamp_exp_arg(u);
  const double tk = fma(u, -kInvStep, kMagic);
  const int kb = __double2loint(tk);  // k (two's complement), k <= 0
  const double kd = tk - kMagic;      // k, exactly
  const double f = fma(kd, -kStep, -u);                              // e^-u = 2^(k/2^BITS) e^f
  double p;
  if constexpr (BITS >= FKTB_EXP_DEG2_BITS) {  // |f| <= ln2/2^11 at BITS = 10: degree 2, truncation <= 6.5e-12
    p = 0.5;
  } else if constexpr (BITS >= 9) {  // |f| <= ln2/2^10: degree 3, truncation <= 9e-15
    p = fma(f, 1.0 / 6.0, 0.5);
  } else {  // |f| <= 0.53 ln2/2^(BITS-1): degree 4, truncation <= 5e-14 at BITS = 6
    p = fma(f, 1.0 / 24.0, 1.0 / 6.0);
    p = fma(f, p, 0.5);
  }
  p = fma(f, p, 1.0);
  p = fma(f, p, 1.0);
  const double tj = exp_table_at<REP, BITS>(tab, kb, colBytes);
  // exponent: the table is stored pre-compensated (expTableDevice(bits,
  // true): entry j's high word minus j << (20 - BITS)), so one shift-add,
  // hi(tj) + (kb << (20 - BITS)), adds floor(k / 2^BITS) << 20 to the true
  // entry's exponent: kb << (20 - BITS) = (e << 20) + (j << (20 - BITS)) mod
  // 2^32 for k = e 2^BITS + j
  const unsigned eh = static_cast<unsigned>(__double2hiint(tj)) + (static_cast<unsigned>(kb) << (20 - BITS));
  return __hiloint2double(static_cast<int>(eh), __double2loint(tj)) * p;
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
