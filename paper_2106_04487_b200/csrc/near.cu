// K3: near field (reference proj/src/transform.cpp:163-181).
//
// For every leaf l and target t in its near set N_l:
//   z_t += sum_{s in l} K(|x_t - x_s|) y_s      (K(0) -> diagonal convention)
// Work tiles are (leaf, <= kNearTile targets of N_l). One CTA stages the
// leaf's sources (SoA coordinates + weights, contiguous in permuted order) in
// shared memory and every thread register-blocks kNearTPT targets against
// broadcast shared-memory reads of the sources. FP64 throughout; the pair
// loop is FP64-pipe bound.
#include "device_math.cuh"
#include "fastmath.cuh"
#include "near_common.cuh"
#include "plan.hpp"

#include <cmath>
#include <cstdlib>
#include <mutex>

namespace fktb {
namespace {

constexpr int kNearThreads = 128;
constexpr int kNearTPT = 2;
constexpr int kNearChunk = 512;  // sources staged per pass (generic kernel)
constexpr int kFastChunk = 512;  // sources staged per pass (fast kernel)
// CTAs/SM hint per kernel (B200 sweep, 64-thread CTAs): Matern-3/2 in 3-D runs
// fastest capped at 10 CTAs (<= 102 registers; cfg2 K3 13.61 -> 13.42 ms);
// the others are best left to ptxas (cfg3/cfg4 slower when capped).
constexpr int nearMinBlocks(int kid, int d) { return kid == FKTB_KERNEL_MATERN32 && d == 3 ? 10 : 1; }

struct NearArgs {
  int n, d, nrhs;
  const double* pc;  // SoA permuted coordinates
  const uint32_t* begin;
  const uint32_t* end;
  const FktbTile* tiles;
  const uint32_t* nearPos;
  const double* yp;  // permuted weights, n x nrhs
  double* zp;        // permuted output, n x nrhs
  FktbKernelDesc kd;
};

template <int KID, int D>
__global__ void __launch_bounds__(kNearThreads) near_kernel(const __grid_constant__ NearArgs A) {
  constexpr int DD = D > 0 ? D : FKTB_MAX_DIM;
  const int d = D > 0 ? D : A.d;
  extern __shared__ double smem[];
  double* sw = smem;                 // [kNearChunk]
  double* sx = smem + kNearChunk;    // [d][kNearChunk]
  const FktbTile tile = A.tiles[blockIdx.x];
  const int leaf = tile.node;
  const int sb = static_cast<int>(A.begin[leaf]), se = static_cast<int>(A.end[leaf]);
  const int n = A.n;

  int tpos[kNearTPT];
  double tx[kNearTPT][DD];
  double acc[kNearTPT];
#pragma unroll
  for (int i = 0; i < kNearTPT; ++i) {
    const int idx = threadIdx.x + i * kNearThreads;
    tpos[i] = idx < tile.count ? static_cast<int>(A.nearPos[tile.start + idx]) : -1;
    const int p = tpos[i] >= 0 ? tpos[i] : 0;
#pragma unroll
    for (int a = 0; a < DD; ++a)
      if (a < d) tx[i][a] = A.pc[static_cast<size_t>(a) * n + p];
    acc[i] = 0.0;
  }
  for (int rhs = 0; rhs < A.nrhs; ++rhs) {
    const double* y = A.yp + static_cast<size_t>(rhs) * n;
    for (int cs = sb; cs < se; cs += kNearChunk) {
      const int cn = min(kNearChunk, se - cs);
      __syncthreads();
      for (int s = threadIdx.x; s < cn; s += kNearThreads) {
        sw[s] = y[cs + s];
        for (int a = 0; a < d; ++a) sx[a * kNearChunk + s] = A.pc[static_cast<size_t>(a) * n + cs + s];
      }
      __syncthreads();
#pragma unroll 2
      for (int s = 0; s < cn; ++s) {
        double sxa[DD];
#pragma unroll
        for (int a = 0; a < DD; ++a)
          if (a < d) sxa[a] = sx[a * kNearChunk + s];
        const double w = sw[s];
#pragma unroll
        for (int i = 0; i < kNearTPT; ++i) {
          double dist2 = 0.0;
#pragma unroll
          for (int a = 0; a < DD; ++a) {
            if (a < d) {
              const double t = tx[i][a] - sxa[a];
              dist2 = fma(t, t, dist2);
            }
          }
          double kv = kernel_value<KID>(A.kd, dist2);
          kv = dist2 == 0.0 ? A.kd.diag : kv;
          acc[i] = fma(kv, w, acc[i]);
        }
      }
    }
    double* z = A.zp + static_cast<size_t>(rhs) * n;
#pragma unroll
    for (int i = 0; i < kNearTPT; ++i) {
      if (tpos[i] >= 0) atomicAdd(z + tpos[i], acc[i]);
      acc[i] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// Fast path for the hot kernels in d = 2, 3, 5: coordinates pre-scaled by the
// kernel length scale (and weights by its prefactor) so the pair body is the
// canonical kernel; FP64 fast math (fastmath.cuh); 4 targets per thread
// against AoS shared-memory sources read with 128-bit broadcast loads.

struct FastArgs {
  NearArgs a;
  double sc, wf;
  double diagCanon;  // diag / wf
  int sel;           // apply the r == 0 convention explicitly
  const double* expTable;
  // Gram-form tiles (kernels with FastKernel::gram, no explicit r == 0
  // select): leaf centres (nodes x d) and limit^2 = (radius/theta)^2; a tile
  // takes the Gram form when limit2[leaf] <= gramLimit2 (scaled |t|^2 + |s|^2
  // <= kGramBound), else the difference form. gramLimit2 < 0 disables it.
  const double* center;
  const double* limit2;
  double gramLimit2;
};

// Bound B on |t|^2 + |s|^2 (scaled, leaf-centred) for the Gram form. Near
// targets of leaf l lie within radius/theta of its centre (tree.cpp:191-200),
// sources within radius, so a tile's B = limit2 * sc^2 * (1 + theta^2). The
// rounding of q is <= ~(4 + d) eps * B absolute (random-walk typical); every
// Gram kernel has |dK/dq| <= 1 in canonical scaling, so K errs by <= ~1e-13
// at B = 128 (cfg2's leaves: B ~ 7). q <= 2B keeps sqrt(q) and the Gaussian's
// exp argument far below the exp clamp (no clamp in the pair body).
constexpr double kGramBound = 128.0;

// FP32-indexed exp (fastmath.cuh exp_neg_fi) in the near field; compile-time
// A/B knob.
#ifndef FKTB_NEAR_FI
#define FKTB_NEAR_FI 1
#endif
constexpr bool kNearFI = FKTB_NEAR_FI != 0;

// Register prefetch of the next shared source row: measured on the B200 at
// cfg2 (Matern d=3) 12.54 -> 12.32 ms and cfg4 (inverse-r d=3) 14.10 -> 13.92,
// but slower for the 5-D Gaussian (21.65 -> 21.96) and 16 RHS (4.16 -> 4.27),
// whose rows are wider: on for single-RHS 3-D tiles. FKTB_NEAR_PF=0/1 forces.
#ifndef FKTB_NEAR_PF
#define FKTB_NEAR_PF -1
#endif
constexpr bool nearPrefetch(int d, int r) { return FKTB_NEAR_PF >= 0 ? FKTB_NEAR_PF != 0 : (d == 3 && r == 1); }

// Runtime A/B knob: FKTB_NEAR_GRAM=0 forces the difference form everywhere.
inline bool nearGramEnabled() {
  static const bool v = [] {
    const char* e = std::getenv("FKTB_NEAR_GRAM");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Shared AoS source rows: stride (doubles, even for 128-bit loads) and the
// sources staged per pass. Gram rows carry |s|^2 too; their chunk is halved to
// keep shared memory (and so occupancy) at the difference form's level; many
// right-hand sides shrink the chunk to stay within 40 KB of static shared
// memory next to the 8 KB exp table.
constexpr int nearStride(int d, int r, bool gram, bool factored = false) {
  return (d + (gram && !factored ? 1 : 0) + r + 1) / 2 * 2;
}
constexpr int nearChunk(int d, int r, bool gram) {
  return gram ? (r > 2 ? 128 : 256) : (r <= 2 ? kFastChunk : (nearStride(d, r, false) * 256 * 8 <= 40960 ? 256 : 128));
}

// Whole tile pass (targets, source chunks, atomics) in one pair form.
//  GRAM = false: q = sum_a (t_a - s_a)^2 on scaled coordinates (bias kQBias),
//    sources AoS (s_0..s_{D-1}, w_0..w_{R-1}).
//  GRAM = true: t, s centred on the leaf centre c; q = |t|^2 + (|s|^2 +
//    offset) + sum_a t_a (-2 s_a), sources AoS (-2 s_a, |s|^2 + offset, w_r):
//    D FMAs + 1 add per pair instead of D subtractions + D FMAs.
template <int KID, int D, bool SEL, int THREADS, int TPT, int UNR, int R, bool GRAM, bool FI>
__device__ __forceinline__ void near_tile(const FastArgs& F, const FktbTile& tile, double* ss, const double* tab,
                                          int colBytes) {
  using FK = FastKernel<KID>;
  constexpr bool FAC = GRAM && FK::gramFactored;
  constexpr int SP = nearStride(D, R, GRAM, FAC);
  constexpr int CHUNK = nearChunk(D, R, GRAM);
  const NearArgs& A = F.a;
  const int leaf = tile.node;
  const int sb = static_cast<int>(A.begin[leaf]), se = static_cast<int>(A.end[leaf]);
  const int n = A.n;
  double c[D];
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = GRAM ? F.center[static_cast<size_t>(leaf) * D + a] : 0.0;
  const double wf = GRAM && !FAC ? F.wf * FK::gramWeight : F.wf;  // weight prefactor of this form
  // factored Gaussian: q = Bt - 2 t.s >= 0 with Bt just above this tile's
  // bound B >= |t|^2 + |s|^2 >= 2 t.s (the 1e-6 and 1e-30 margins cover the
  // rounding and keep q >= 2^-127 for the FP32-indexed exp); q <= 2.1 B
  const double Bt = FAC ? fma(1.000001 * kGramBound / F.gramLimit2, F.limit2[leaf], 1e-30) : 0.0;
  // Matern's Gram bias: q's rounding is <= (1.5 d + 0.5) eps B for this tile's
  // B = limit2 * kGramBound / gramLimit2 (|t|^2, |s|^2: d/2 eps B each; d FMAs
  // and one add: (d + 1)/2 eps B), so q + (1.5 d + 1) eps B + 1e-30 >= 1e-30
  // without a clamp; it shifts K by <= half of it (|dK/dq| <= 1/2): ~3e-15 at
  // cfg2's B ~ 7, 5e-14 at B = 70
  const double qbias = GRAM && FK::gramBiased
                           ? fma((1.5 * D + 1.0) * 2.220446049250313e-16 * kGramBound / F.gramLimit2, F.limit2[leaf], 1e-30)
                           : 0.0;
  int tpos[TPT];
  double tx[TPT][D];
  double tn[TPT];
  double acc[TPT][R];
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    const int idx = threadIdx.x + i * THREADS;
    tpos[i] = idx < tile.count ? static_cast<int>(A.nearPos[tile.start + idx]) : -1;
    const int p = tpos[i] >= 0 ? tpos[i] : 0;
    tn[i] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if constexpr (GRAM) {
        tx[i][a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + p] - c[a], F.sc);
        tn[i] = fma(tx[i][a], tx[i][a], tn[i]);
      } else {
        // __dmul_rn: never contracted into the pair loop's subtraction, so a
        // target and a source at the same point scale to the same double and
        // r == 0 gives q == kQBias exactly (the select depends on it)
        tx[i][a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + p], F.sc);
      }
    }
  }
  for (int r0 = 0; r0 < A.nrhs; r0 += R) {
#pragma unroll
    for (int i = 0; i < TPT; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
    for (int cs = sb; cs < se; cs += CHUNK) {
      const int cn = min(CHUNK, se - cs);
      __syncthreads();
      for (int s = threadIdx.x; s < cn; s += THREADS) {
        if constexpr (GRAM) {
          double ns = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double v = __dmul_rn(A.pc[static_cast<size_t>(a) * n + cs + s] - c[a], F.sc);
            ns = fma(v, v, ns);
            ss[s * SP + a] = -2.0 * v;
          }
          if constexpr (FAC) {
            const double ef = wf * exp(Bt - ns);  // e^(B - |s|^2) in [1, e^B]
#pragma unroll
            for (int r = 0; r < R; ++r) ss[s * SP + D + r] = A.yp[static_cast<size_t>(r0 + r) * n + cs + s] * ef;
          } else {
            ss[s * SP + D] = ns + (FK::gramOffset + qbias);
#pragma unroll
            for (int r = 0; r < R; ++r) ss[s * SP + D + 1 + r] = A.yp[static_cast<size_t>(r0 + r) * n + cs + s] * wf;
          }
        } else {
#pragma unroll
          for (int a = 0; a < D; ++a) ss[s * SP + a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + cs + s], F.sc);
#pragma unroll
          for (int r = 0; r < R; ++r) ss[s * SP + D + r] = A.yp[static_cast<size_t>(r0 + r) * n + cs + s] * F.wf;
        }
      }
      __syncthreads();
      constexpr int W0 = GRAM && !FAC ? D + 1 : D;  // first weight slot
      // the pair block of one source row against this thread's TPT targets
      auto pairs = [&](const double(&src)[SP]) {
#pragma unroll
        for (int i = 0; i < TPT; ++i) {
          double q;
          if constexpr (FAC) {
            q = fma(tx[i][0], src[0], Bt);
#pragma unroll
            for (int a = 1; a < D; ++a) q = fma(tx[i][a], src[a], q);
          } else if constexpr (GRAM) {
            q = fma(tx[i][0], src[0], src[D]);
#pragma unroll
            for (int a = 1; a < D; ++a) q = fma(tx[i][a], src[a], q);
            q += tn[i];
          } else {
            const double d0 = tx[i][0] - src[0];
            q = fma(d0, d0, kQBias);
#pragma unroll
            for (int a = 1; a < D; ++a) {
              const double da = tx[i][a] - src[a];
              q = fma(da, da, q);
            }
          }
          double kv = FK::template eval<kNearExpRep, FI, GRAM>(q, tab, colBytes);
          // r == 0 <=> q == kQBias; compared on the high word (integer pipe):
          // any other q is >= ~1e-284 (points closer than ~1e-142 count as
          // coincident, where the FP64 form was already off)
          if constexpr (SEL) kv = __double2hiint(q) == kQBiasHi ? F.diagCanon : kv;
#pragma unroll
          for (int r = 0; r < R; ++r) acc[i][r] = fma(kv, src[W0 + r], acc[i][r]);
        }
      };
      auto load = [&](double(&src)[SP], int s) {
#pragma unroll
        for (int q = 0; q < SP; q += 2) {
          const double2 v = *reinterpret_cast<const double2*>(&ss[s * SP + q]);
          src[q] = v.x;
          src[q + 1] = v.y;
        }
      };
      if constexpr (nearPrefetch(D, R)) {
        // software pipeline: row s + 1 is loaded while row s is evaluated (the
        // broadcast LDS latency otherwise stalls the first FMA of every row);
        // row cn is a padding row of the shared array, loaded but never used
        double cur[SP];
        load(cur, 0);
#pragma unroll UNR
        for (int s = 0; s < cn; ++s) {
          double nxt[SP];
          load(nxt, s + 1);
          pairs(cur);
#pragma unroll
          for (int q = 0; q < SP; ++q) cur[q] = nxt[q];
        }
      } else {
#pragma unroll UNR
        for (int s = 0; s < cn; ++s) {
          double src[SP];
          load(src, s);
          pairs(src);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TPT; ++i)
      if (tpos[i] >= 0) {
        const double tf = FAC ? exp(-tn[i]) : 1.0;  // factored Gaussian: e^-|t|^2
#pragma unroll
        for (int r = 0; r < R; ++r) atomicAdd(A.zp + static_cast<size_t>(r0 + r) * n + tpos[i], FAC ? acc[i][r] * tf : acc[i][r]);
      }
  }
}

// THREADS x TPT = 256 targets per tile; UNR sources per unrolled step; R
// right-hand sides per pass (the kernel value is evaluated once per pair and
// reused for all R weights). GRAM: this launch serves the tiles whose leaf
// passes the Gram bound (the other launch, GRAM = false, the rest); separate
// instantiations so each form gets its own register allocation.
// MB: CTAs/SM for __launch_bounds__ (0: nearMinBlocks for 64-thread single-RHS
// shapes, else none).
template <int KID, int D, bool SEL, int THREADS, int TPT, int UNR, int R, bool GRAM, int MB>
__global__ void __launch_bounds__(THREADS, (MB > 0 ? MB : (THREADS == 64 && R == 1 ? nearMinBlocks(KID, D) : 1))) near_fast(const __grid_constant__ FastArgs F) {
  static_assert(THREADS * TPT == kNearThreads * kNearTPT, "near tile size");
  static_assert(!GRAM || (FastKernel<KID>::gram && !SEL), "Gram form needs a smooth kernel without select");
  constexpr int SP = nearStride(D, R, GRAM);
  constexpr int CHUNK = nearChunk(D, R, GRAM);
  __shared__ __align__(16) double ss[(CHUNK + 1) * SP];  // + a padding row for the prefetch
  __shared__ double tab[kNearExpTable * kNearExpRep];  // entry j at tab[j * kNearExpRep + column]
  const NearArgs& A = F.a;
  const FktbTile tile = A.tiles[blockIdx.x];
  if (GRAM != (F.limit2[tile.node] <= F.gramLimit2)) return;  // the other form's tile
  if constexpr (FastKernel<KID>::needsTable)
    for (int i = threadIdx.x; i < kNearExpTable * kNearExpRep; i += THREADS) tab[i] = F.expTable[i / kNearExpRep];
  // each lane reads its own column: conflict-free 64-bit lookups
  near_tile<KID, D, SEL, THREADS, TPT, UNR, R, GRAM, kNearFI>(F, tile, ss, tab, (threadIdx.x & (kNearExpRep - 1)) * 8);
}

template <int KID, int D, bool SEL, int THREADS, int TPT, int UNR, int R, int MB = 0>
void launchFastV(const FastArgs& F, int tiles, int gramTiles, cudaStream_t st) {
  if constexpr (FastKernel<KID>::gram && !SEL) {
    if (gramTiles > 0) {
      near_fast<KID, D, SEL, THREADS, TPT, UNR, R, true, MB><<<tiles, THREADS, 0, st>>>(F);
      FKTB_CUDA(cudaGetLastError());
    }
  } else {
    gramTiles = 0;
  }
  if (gramTiles < tiles) {
    near_fast<KID, D, SEL, THREADS, TPT, UNR, R, false, MB><<<tiles, THREADS, 0, st>>>(F);
    FKTB_CUDA(cudaGetLastError());
  }
}

template <int KID, int D, bool SEL>
void launchFastSel(const FastArgs& F, int nrhs, int tiles, int gramTiles, cudaStream_t st) {
  if (nrhs == 1) {
    // measured shapes (B200 sweeps of the round-1 shape knob): Matern-3/2 in 3-D
    // wants 8 independent targets per thread (one warp per CTA: cfg2 K3
    // 13.72 -> 13.14 ms before the clamp-free Gram form, tied with 64 x 4
    // after it); the 5-D Gaussian 8 CTAs/SM (cfg3 22.6 -> 21.7 ms)
    if constexpr (KID == FKTB_KERNEL_MATERN32 && D == 3 && !SEL) return launchFastV<KID, D, SEL, 32, 8, 2, 1>(F, tiles, gramTiles, st);
    if constexpr (KID == FKTB_KERNEL_GAUSSIAN && D == 5 && !SEL) return launchFastV<KID, D, SEL, 64, 4, 2, 1, 8>(F, tiles, gramTiles, st);
    return launchFastV<KID, D, SEL, 64, 4, 2, 1>(F, tiles, gramTiles, st);
  }
  if (nrhs % 16 == 0) {
    // 4 targets x 16 RHS accumulators per thread: each source's 16 weights
    // (8 LDS.128) serve 64 FMAs (cfg5 K3 4.95 -> 4.21 ms vs 1 target/thread)
    return launchFastV<KID, D, SEL, 64, 4, 1, 16>(F, tiles, gramTiles, st);
  }
  if (nrhs % 8 == 0) return launchFastV<KID, D, SEL, 128, 2, 2, 8>(F, tiles, gramTiles, st);
  if (nrhs % 4 == 0) return launchFastV<KID, D, SEL, 128, 2, 2, 4>(F, tiles, gramTiles, st);
  if (nrhs % 2 == 0) return launchFastV<KID, D, SEL, 64, 4, 2, 2>(F, tiles, gramTiles, st);
  return launchFastV<KID, D, SEL, 64, 4, 2, 1>(F, tiles, gramTiles, st);
}

// Tiles whose leaf passes the Gram bound: the device test, on the same limit2
// values (tree.cu computes limit2 the same way).
long long countGramTiles(const DevicePlan& plan, double gramLimit2) {
  const DeviceTree& t = *plan.tree;
  long long g = 0;
  for (const FktbTile& tl : plan.nearTilesHost) {
    volatile double limit = t.radius[static_cast<size_t>(tl.node)] / t.theta;
    g += limit * limit <= gramLimit2;
  }
  return g;
}

template <int KID, int D>
void launchFastT(const NearArgs& A, const DevicePlan& plan, int tiles, cudaStream_t st) {
  const DeviceTree& t = *plan.tree;
  FastArgs F{A, 1.0, 1.0, 0.0, 0, expTableDevice(kNearExpBits), t.dCenter.get(), t.dLimit2.get(), -1.0};
  fastScales(A.kd, F.sc, F.wf);
  F.diagCanon = A.kd.diag / F.wf;
  // The canonical formula already gives the reference convention at r == 0
  // for the smooth kernels (K(0) = valueAtZero); otherwise select explicitly.
  const bool smooth = KID != FKTB_KERNEL_INVERSE_R && KID != FKTB_KERNEL_INVERSE_R2;
  F.sel = !(smooth && A.kd.diag == F.wf);
  // Gram tiles only without the select (it needs exact r == 0 detection);
  // gramLimit2 < 0 leaves every tile to the difference form.
  int gramTiles = 0;
  if (FastKernel<KID>::gram && !F.sel && nearGramEnabled()) {
    F.gramLimit2 = kGramBound / (F.sc * F.sc * (1.0 + t.theta * t.theta));
    gramTiles = static_cast<int>(countGramTiles(plan, F.gramLimit2));
  }
  if (F.sel)
    launchFastSel<KID, D, true>(F, A.nrhs, tiles, gramTiles, st);
  else
    launchFastSel<KID, D, false>(F, A.nrhs, tiles, gramTiles, st);
}

template <int KID, int D>
void launchNearT(const NearArgs& A, int tiles, cudaStream_t st) {
  const int d = D > 0 ? D : A.d;
  const size_t smem = static_cast<size_t>(kNearChunk) * (d + 1) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    FKTB_CUDA(cudaFuncSetAttribute(near_kernel<KID, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kNearChunk * (FKTB_MAX_DIM + 1) * sizeof(double))));
    configured = true;
  }
  near_kernel<KID, D><<<tiles, kNearThreads, smem, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

template <int KID>
void launchNearK(const NearArgs& A, const DevicePlan& plan, int tiles, cudaStream_t st) {
  if constexpr (FastKernel<KID>::supported) {
    switch (A.d) {
      case 2: return launchFastT<KID, 2>(A, plan, tiles, st);
      case 3: return launchFastT<KID, 3>(A, plan, tiles, st);
      case 5: return launchFastT<KID, 5>(A, plan, tiles, st);
      default: break;
    }
  }
  switch (A.d) {
    case 2: return launchNearT<KID, 2>(A, tiles, st);
    case 3: return launchNearT<KID, 3>(A, tiles, st);
    case 5: return launchNearT<KID, 5>(A, tiles, st);
    default: return launchNearT<KID, 0>(A, tiles, st);
  }
}

}  // namespace

// 2^(j/2^bits), j < 2^bits, correctly rounded (host long double); one table
// per size, built once (outside any graph capture: see createPlan).
const double* expTableDevice(int bits) {
  static double* dev[16] = {};
  static std::once_flag once[16];
  if (bits < 0 || bits >= 16) throw std::invalid_argument("exp table size");
  std::call_once(once[bits], [bits] {
    const int n = 1 << bits;
    std::vector<double> host(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) host[static_cast<size_t>(j)] = static_cast<double>(std::exp2(static_cast<long double>(j) / n));
    FKTB_CUDA(cudaMalloc(&dev[bits], host.size() * sizeof(double)));
    FKTB_CUDA(cudaMemcpy(dev[bits], host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice));
  });
  return dev[bits];
}

int nearTileSize() { return kNearThreads * kNearTPT; }

// Gram-form tiles of the FP64 near_fast launch (0 when the plan's kernel,
// dimension or diagonal convention keeps the difference form); mirrors the
// decisions of launchFastT.
long long nearGramTiles(const DevicePlan& plan) {
  const int d = plan.tree->d;
  if (d != 2 && d != 3 && d != 5) return 0;
  const int id = plan.kernel.id;
  const bool gram = id == FKTB_KERNEL_MATERN32 || id == FKTB_KERNEL_CAUCHY || id == FKTB_KERNEL_RATIONAL_QUADRATIC ||
                    id == FKTB_KERNEL_GAUSSIAN;
  if (!gram || !nearGramEnabled()) return 0;
  FktbKernelDesc kd;
  fillKernelDesc(plan.kernel, kd);
  if (plan.options.hasDiagonal) kd.diag = plan.options.diagonal;
  double sc, wf;
  fastScales(kd, sc, wf);
  if (kd.diag != wf) return 0;  // explicit r == 0 select
  const DeviceTree& t = *plan.tree;
  return countGramTiles(plan, kGramBound / (sc * sc * (1.0 + t.theta * t.theta)));
}

void launchNear(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t st) {
  const int tiles = static_cast<int>(plan.nearTilesHost.size());
  if (tiles == 0) return;
  const DeviceTree& t = *plan.tree;
  NearArgs A{t.n, t.d, nrhs, t.pc.get(), t.dBegin.get(), t.dEnd.get(), plan.dNearTiles.get(), t.dNearPos.get(), yp, zp, {}};
  fillKernelDesc(plan.kernel, A.kd);
  if (plan.options.hasDiagonal) A.kd.diag = plan.options.diagonal;
  switch (plan.kernel.id) {
    case FKTB_KERNEL_EXPONENTIAL: return launchNearK<FKTB_KERNEL_EXPONENTIAL>(A, plan, tiles, st);
    case FKTB_KERNEL_MATERN12: return launchNearK<FKTB_KERNEL_MATERN12>(A, plan, tiles, st);
    case FKTB_KERNEL_MATERN32: return launchNearK<FKTB_KERNEL_MATERN32>(A, plan, tiles, st);
    case FKTB_KERNEL_CAUCHY: return launchNearK<FKTB_KERNEL_CAUCHY>(A, plan, tiles, st);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return launchNearK<FKTB_KERNEL_RATIONAL_QUADRATIC>(A, plan, tiles, st);
    case FKTB_KERNEL_GAUSSIAN: return launchNearK<FKTB_KERNEL_GAUSSIAN>(A, plan, tiles, st);
    case FKTB_KERNEL_INVERSE_R: return launchNearK<FKTB_KERNEL_INVERSE_R>(A, plan, tiles, st);
    case FKTB_KERNEL_INVERSE_R2: return launchNearK<FKTB_KERNEL_INVERSE_R2>(A, plan, tiles, st);
    case FKTB_KERNEL_INVERSE_R3: return launchNearK<FKTB_KERNEL_INVERSE_R3>(A, plan, tiles, st);
    case FKTB_KERNEL_EXP_OVER_R: return launchNearK<FKTB_KERNEL_EXP_OVER_R>(A, plan, tiles, st);
    case FKTB_KERNEL_R_EXP: return launchNearK<FKTB_KERNEL_R_EXP>(A, plan, tiles, st);
    case FKTB_KERNEL_COS_OVER_R: return launchNearK<FKTB_KERNEL_COS_OVER_R>(A, plan, tiles, st);
    case FKTB_KERNEL_EXP_NEG_INV_R: return launchNearK<FKTB_KERNEL_EXP_NEG_INV_R>(A, plan, tiles, st);
    case FKTB_KERNEL_EXP_NEG_INV_R2: return launchNearK<FKTB_KERNEL_EXP_NEG_INV_R2>(A, plan, tiles, st);
  }
  throw std::invalid_argument("near field: unknown kernel id");
}

}  // namespace fktb
