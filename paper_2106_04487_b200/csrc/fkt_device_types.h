// POD descriptors shared by the host plan code and the sm_100a kernels.
// Plain C layout: these travel as CUDA kernel parameters (constant bank 0,
// __grid_constant__), so every per-pair table lookup with a compile-time index
// becomes an immediate constant-bank operand.
#ifndef FKTB_DEVICE_TYPES_H
#define FKTB_DEVICE_TYPES_H

#include <stdint.h>

#define FKTB_MAX_DIM 16
#define FKTB_MAX_P 20
#define FKTB_TBAR_CAP 1760   // sum_{k<=p, j=k,k+2..p} j  at p = 20 is 1650
#define FKTB_FACTOR_CAP 1400 // compressed factor coefficients (target + source)
#define FKTB_FACTOR_MAX 128  // number of (k, i) factors: sum_k rank_k <= 121 at p = 20

// Built-in kernels, in reference proj/src/kernels.cpp:158-160 order.
enum {
  FKTB_KERNEL_EXPONENTIAL = 0,
  FKTB_KERNEL_MATERN12 = 1,
  FKTB_KERNEL_MATERN32 = 2,
  FKTB_KERNEL_CAUCHY = 3,
  FKTB_KERNEL_RATIONAL_QUADRATIC = 4,
  FKTB_KERNEL_GAUSSIAN = 5,
  FKTB_KERNEL_INVERSE_R = 6,
  FKTB_KERNEL_INVERSE_R2 = 7,
  FKTB_KERNEL_INVERSE_R3 = 8,
  FKTB_KERNEL_EXP_OVER_R = 9,
  FKTB_KERNEL_R_EXP = 10,
  FKTB_KERNEL_COS_OVER_R = 11,
  FKTB_KERNEL_EXP_NEG_INV_R = 12,
  FKTB_KERNEL_EXP_NEG_INV_R2 = 13,
  FKTB_KERNEL_COUNT = 14
};

typedef struct FktbKernelDesc {
  int id;
  int pad_;
  double s2;    // sigma^2 (matern12/32)
  double a;     // sqrt(3)/rho (matern32)
  double is2;   // 1/sigma^2 (cauchy, rational-quadratic)
  double rho;   // matern12 length scale
  double diag;  // value used at r == 0 (override, else the kernel's convention)
} FktbKernelDesc;

// Far-field (s2m / m2t) expansion description for one plan.
typedef struct FktbFarParams {
  int d, p;
  int P;   // coefficients per node (layout total)
  int H;   // harmonics of degree <= p
  int compressed;
  int pad_;
  FktbKernelDesc kernel;
  int Pref;  // the reference layout total (coefficientCount(); compressed ranks)
  int hOff[FKTB_MAX_P + 2];     // first harmonic of degree k
  // Stored moment layout is always the padded uncompressed one (degree-major,
  // harmonic, slot with slotsU[k] = (p-k)/2+1 slots); compressed plans fill
  // only the first slots[k] = rank_k of them. P above is the padded total.
  int cOff[FKTB_MAX_P + 2];     // first coefficient of degree k
  int slotsU[FKTB_MAX_P + 1];   // (p-k)/2 + 1
  int slots[FKTB_MAX_P + 1];    // used slots (uncompressed slotsU[k], else rank_k)
  // Uncompressed radial table: for (k, slot s), j = k + 2s, entries m = 1..j of
  // Tbar_kjm * m! (reference coefficients.cpp:52-95, expansion.cpp:27-40).
  int tOff[FKTB_MAX_P + 2];     // first (k, s) row of degree k: sum_{k'<k} slotsU[k']
  int tRow[FKTB_MAX_P * FKTB_MAX_P];  // row start in tb, indexed tOff[k] + s
  double tb[FKTB_TBAR_CAP];
  // Compressed factors (reference expansion.cpp:190-243): factor f = fOff[k]+i
  // target Laurent sum_{e=fLo..fHi} fc[fAt[f] + e - fLo] r^e (multiplies K(r)),
  // source polynomial sum_{e=gLo..gHi} fc[gAt[f] + e - gLo] r'^e.
  // Dense target-factor windows (compile-time exponent range per kernel, see
  // compressed_window in device_math.cuh): factor f, power e in [denseLo,
  // denseHi] at fc[denseAt + f * (denseHi - denseLo + 1) + e - denseLo];
  // denseAt < 0 when the factors do not fit (runtime loops are used then).
  int denseLo, denseHi, denseAt;
  int fOff[FKTB_MAX_P + 2];
  int fLo[FKTB_FACTOR_MAX], fHi[FKTB_FACTOR_MAX], fAt[FKTB_FACTOR_MAX];
  int gLo[FKTB_FACTOR_MAX], gHi[FKTB_FACTOR_MAX], gAt[FKTB_FACTOR_MAX];
  double fc[FKTB_FACTOR_CAP];
} FktbFarParams;

// Runtime harmonic chain table for the generic (runtime d, p) kernels:
// harmonic h = gIdx[h*(d-2) + level-1] into the per-level Gegenbauer table,
// circular index cIdx[h], phase ph[h] (+1 cos / -1 sin / 0).
typedef struct FktbChainTable {
  const int* gIdx;
  const int* cIdx;
  const int* ph;
} FktbChainTable;

// Work tile: targets [start, start+count) of list `node`.
typedef struct FktbTile {
  int node;
  int count;
  int64_t start;
} FktbTile;

#endif
