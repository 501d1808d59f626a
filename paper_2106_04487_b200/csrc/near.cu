// K3: near field (reference proj/src/transform.cpp:163-181).
//
// For every leaf l and target t in its near set N_l:
//   z_t += sum_{s in l} K(|x_t - x_s|) y_s      (K(0) -> diagonal convention)
// Work tiles are (leaf, <= 256 targets of N_l). The hot kernels in d = 2, 3,
// 5 run the persistent TMA-fed near_stream (below); every other (kernel, d)
// the generic near_kernel, which stages the leaf's sources in shared memory
// per CTA. FP64 throughout; the pair loop is FP64-pipe bound.
#include "device_math.cuh"
#include "fastmath.cuh"
#include "near_common.cuh"
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace fktb {
namespace {

constexpr int kNearTileTargets = 256;  // targets per work tile (both paths)
constexpr int kNearThreads = 128;      // generic kernel: 128 threads x 2 targets
constexpr int kNearTPT = 2;
constexpr int kNearChunk = 512;  // sources staged per pass (generic kernel)

struct NearArgs {
  int n, d, nrhs;
  const double* pc;  // SoA permuted coordinates
  const uint32_t* begin;
  const uint32_t* end;
  const FktbTile* tiles;
  const uint32_t* nearPos;
  const double* yp;  // permuted weights, n x nrhs
  ZOut out;          // permuted output, n x nrhs (atomics or deterministic slots)
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
#pragma unroll
    for (int i = 0; i < kNearTPT; ++i) {
      if (tpos[i] >= 0) A.out.add(rhs, tile.start + threadIdx.x + i * kNearThreads, tpos[i], acc[i]);
      acc[i] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// Fast path for the hot kernels in d = 2, 3, 5: a persistent, TMA-fed kernel.
//
//  * Geometry rows (plan time, near_rows_kernel): per source position p, GS
//    doubles in HBM: Gram leaves (-2g s~_a, g (|s~|^2 +
//    offset + bias)), factored Gram (-2 s~_a), difference leaves (s~_a), with
//    s~ = (x - c_leaf) sc or x sc; g = FastKernel::gramScale.
//  * Weights (per multiply): y in tree order (yp) for one RHS, else a
//    source-major copy of the pass's R columns (near_weights_kernel; the
//    factored Gaussian's per-source factor folded in).
//  * Work tiles (leaf, <= 256 targets of its near list), Gram tiles first;
//    one launch per pair form. Persistent one-warp CTAs claim (tile, part)
//    work units; every lane register-blocks TPT targets. The leaf's
//    source rows stream through a two-stage shared-memory ring: one thread
//    arms an mbarrier with the byte count and issues cp.async.bulk for the
//    next chunk (geometry + weights, possibly of the next tile) before the
//    CTA evaluates the current one.
//  * z: one atomic per (target, RHS) per tile, scaled by the constant weight
//    prefactor (FP64 fast math in the pair body: fastmath.cuh).

// Bound B on |t|^2 + |s|^2 (scaled, leaf-centred) for the Gram form. Near
// targets of leaf l lie within radius/theta of its centre (tree.cpp:191-200),
// sources within radius, so a tile's B = limit2 * sc^2 * (1 + theta^2). The
// rounding of q is <= ~(4 + d) eps * B absolute (random-walk typical); every
// Gram kernel has |dK/dq| <= 1 in canonical scaling, so K errs by <= ~1e-13
// at B = 128 (cfg2's leaves: B ~ 7). q <= 2B keeps sqrt(q) and the Gaussian's
// exp argument far below the exp clamp (no clamp in the pair body).
constexpr double kGramBound = 128.0;

// Source row stride (doubles, even: 16-byte rows for the bulk copies): the
// geometry of the kernel's forms (D coordinates, + |s|^2 for the unfactored
// Gram form) and, in the LAST slot, the single-RHS weight (written per
// multiply by near_fill_weights; passes of R > 1 columns read a separate
// source-major weight buffer of stride nearWStride(R)).
template <int KID>
constexpr int nearRowStride(int d) {
  return (d + 1 + (FastKernel<KID>::gram && !FastKernel<KID>::gramFactored ? 1 : 0) + 1) / 2 * 2;
}
constexpr int nearWStride(int r) { return r == 1 ? 0 : (r + 1) / 2 * 2; }

// Register prefetch of the next shared source row: measured on the B200 (round
// 1) at cfg2 (Matern d=3) 12.54 -> 12.32 ms and cfg4 (inverse-r d=3) 14.10 ->
// 13.92, but slower for the 5-D Gaussian and 16 RHS, whose rows are wider: on
// for single-RHS 3-D tiles.
#ifndef FKTB_NEAR_PREFETCH
#define FKTB_NEAR_PREFETCH 1
#endif
constexpr bool nearPrefetch(int d, int r) { return FKTB_NEAR_PREFETCH && d == 3 && r == 1; }

// ---- plan time: geometry rows --------------------------------------------
struct RowArgs {
  int n;
  const double* pc;
  const uint32_t* begin;
  const uint32_t* end;
  const int* left;
  const double* center;
  const double* limit2;
  const unsigned char* leafGram;  // per node: 1 = Gram-form leaf
  double sc, gramLimit2;
  double* rows;  // n x GS
  double* fac;   // factored Gaussian: e^(Bt - |s~|^2) per source (else unused)
};

template <int KID, int D>
__global__ void near_rows_kernel(const __grid_constant__ RowArgs A) {
  using FK = FastKernel<KID>;
  constexpr int GS = nearRowStride<KID>(D);
  constexpr bool FAC = FK::gramFactored;
  const int leaf = blockIdx.x;
  if (A.left[leaf] >= 0) return;
  const bool gram = A.leafGram[leaf] != 0;
  double c[D];
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = gram ? A.center[static_cast<size_t>(leaf) * D + a] : 0.0;
  // Matern's Gram bias: q's rounding is <= (1.5 d + 0.5) eps B for this leaf's
  // B = limit2 * kGramBound / gramLimit2 (|t|^2, |s|^2: d/2 eps B each; d FMAs
  // and one add: (d + 1)/2 eps B), so q + (1.5 d + 1) eps B + 1e-30 >= 1e-30
  // without a clamp; it shifts K by <= half of it (|dK/dq| <= 1/2): ~3e-15 at
  // cfg2's B ~ 7, 5e-14 at B = 70
  const double qbias = gram && FK::gramBiased
                           ? fma((1.5 * D + 1.0) * 2.220446049250313e-16 * kGramBound / A.gramLimit2, A.limit2[leaf], 1e-30)
                           : 0.0;
  // factored Gaussian: q = Bt - 2 t.s >= 0 with Bt just above this leaf's
  // bound B >= |t|^2 + |s|^2 >= 2 t.s (the 1e-6 and 1e-30 margins cover the
  // rounding); q <= 2.1 B
  const double Bt = gram && FAC ? fma(1.000001 * kGramBound / A.gramLimit2, A.limit2[leaf], 1e-30) : 0.0;
  const int sb = static_cast<int>(A.begin[leaf]), se = static_cast<int>(A.end[leaf]);
  for (int p = sb + static_cast<int>(threadIdx.x); p < se; p += blockDim.x) {
    double* row = A.rows + static_cast<size_t>(p) * GS;
    double v[D], ns = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      // __dmul_rn: never contracted, so a target and a source at the same
      // point scale to the same double (difference form: r == 0 gives q ==
      // kQBias exactly, which the select depends on)
      v[a] = __dmul_rn(A.pc[static_cast<size_t>(a) * A.n + p] - c[a], A.sc);
      ns = fma(v[a], v[a], ns);
    }
#pragma unroll
    for (int a = 0; a < GS; ++a) row[a] = 0.0;
    // factored Gaussian: per-source weight factor e^(B - |s|^2) in [1, e^B]
    // on its Gram leaves, 1 on difference-form leaves
    if (FAC && A.fac) A.fac[p] = gram ? exp(Bt - ns) : 1.0;
    if (gram) {
#pragma unroll
      for (int a = 0; a < D; ++a) row[a] = (FAC ? -2.0 : -2.0 * FK::gramScale) * v[a];
      if constexpr (!FAC) row[D] = FK::gramScale * (ns + (FK::gramOffset + qbias));
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) row[a] = v[a];
    }
  }
}

// ---- per multiply: weights ------------------------------------------------
// one RHS: the weight slot of every source row (times the factored Gaussian's
// per-source factor)
__global__ void near_fill_weights(const double* __restrict__ yp, const double* __restrict__ fac,
                                  double* __restrict__ rows, int n, int gs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  rows[static_cast<size_t>(p) * gs + gs - 1] = fac ? yp[p] * fac[p] : yp[p];
}

// R > 1 columns: source-major copy of the pass
__global__ void near_weights_kernel(const double* __restrict__ yp, const double* __restrict__ fac,
                                    double* __restrict__ w, int n, int R, int RP) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double f = fac ? fac[p] : 1.0;
  double* row = w + static_cast<size_t>(p) * RP;
  for (int r = 0; r < RP; r += 2) {
    const double a = yp[static_cast<size_t>(r) * n + p] * f;
    const double b = r + 1 < R ? yp[static_cast<size_t>(r + 1) * n + p] * f : 0.0;
    if (RP == 1) {
      row[0] = a;
    } else {
      *reinterpret_cast<double2*>(row + r) = make_double2(a, b);
    }
  }
}

// ---- the streaming kernel -------------------------------------------------
struct StreamArgs {
  int n;
  const double* pc;  // SoA permuted coordinates (targets)
  const uint32_t* begin;
  const uint32_t* end;
  const FktbTile* tiles;
  int tile0, tile1;  // this launch's tiles [tile0, tile1)
  const uint32_t* nearPos;
  const double* rows;  // source rows, n x GS (single-RHS weight in the last slot)
  const double* w;     // R > 1: source-major weights, n x RP
  ZOut out;            // permuted output, n per RHS (this pass's first column)
  const double* center;
  const double* limit2;
  double sc;         // coordinate scale
  double scale;      // z += scale * acc (the kernel's weight prefactor)
  double diagCanon;  // r == 0 value in canonical units (select)
  double gramLimit2;
  const double* expTable;  // pre-compensated 2^(j/512)
  int* counter;            // tile claims of this launch (zeroed before it)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Sources per pipeline stage: ~10 KB of rows per stage (two stages per
// one-warp CTA, 8-16 CTAs per SM).
#ifndef FKTB_NEAR_STAGE_BYTES
#define FKTB_NEAR_STAGE_BYTES 10240
#endif
constexpr int nearChunk(int gs, int rp) {
  const int c = FKTB_NEAR_STAGE_BYTES / ((gs + rp) * 8);
  return c >= 256 ? 256 : c >= 128 ? 128 : c >= 64 ? 64 : 32;
}

template <int GS, int RP, int CH, bool TAB>
struct NearSmem {
  static constexpr int kGeo = (CH + 1) * GS;  // + the prefetch padding row
  static constexpr int kW = CH * RP;
  static constexpr int kStage = kGeo + kW;    // doubles per stage
  static constexpr int kTab = TAB ? kNearExpTable : 0;
  static constexpr size_t bytes = 16 + sizeof(double) * (kTab + 2 * kStage);
};

// Launch bounds: min CTAs per SM for the shapes that want a register cap
// (round-1 B200 sweeps: the 5-D Gaussian at 16 resident warps per SM).
// (build-time sweep knob for the Matern-3/2 3-D shape: FKTB_NEAR_MINB_M32)
#ifndef FKTB_NEAR_MINB_M32
#define FKTB_NEAR_MINB_M32 1
#endif
#ifndef FKTB_NEAR_G5_TPT
#define FKTB_NEAR_G5_TPT 4   // targets per lane, 5-D Gaussian (sweep knob)
#endif
#ifndef FKTB_NEAR_G5_MINB
#define FKTB_NEAR_G5_MINB 12  // B200 sweep (1024-entry exp table): 8-12 -> 17.03 ms at cfg3, 14-16 -> 18.36
#endif
constexpr int nearMinBlocks(int kid, int d, int r) {
  return kid == FKTB_KERNEL_GAUSSIAN && d == 5 && r == 1 ? FKTB_NEAR_G5_MINB
         : kid == FKTB_KERNEL_MATERN32 && d == 3 && r == 1 ? FKTB_NEAR_MINB_M32
                                                          : 1;
}
#ifndef FKTB_NEAR_UNROLL
#define FKTB_NEAR_UNROLL 2
#endif
constexpr int kNearUnroll = FKTB_NEAR_UNROLL;  // source rows per unrolled step

// One warp per CTA (no CTA-wide barriers: a two-warp version spent 17% of
// their cycles in the per-chunk barrier at cfg4). Work units are (tile, part):
// a tile's 256 targets in 256 / (32 TPT) parts, each streaming the leaf's
// rows on its own (the re-reads hit L2).
template <int KID, int D, bool SEL, int TPT, int R, bool GRAM>
__global__ void __launch_bounds__(32, nearMinBlocks(KID, D, R)) near_stream(const __grid_constant__ StreamArgs A) {
  using FK = FastKernel<KID>;
  static_assert(!GRAM || (FK::gram && !SEL), "Gram form needs a smooth kernel without select");
  constexpr bool FAC = GRAM && FK::gramFactored;
  constexpr int GS = nearRowStride<KID>(D), RP = nearWStride(R);
  constexpr int CH = nearChunk(GS, RP);
  using SM = NearSmem<GS, RP, CH, FK::needsTable>;
  constexpr int PARTS = kNearTileTargets / (32 * TPT);
  static_assert(PARTS * 32 * TPT == kNearTileTargets, "parts must tile the 256 targets");
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw);                   // [2]
  double* tab = reinterpret_cast<double*>(smraw + 16);                  // [kTab]
  double* stage0 = tab + SM::kTab;                                      // [2][kStage]
  const int n = A.n;
  const int lane = threadIdx.x;

  if (threadIdx.x == 0) {
    mbar_init(bar + 0, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (FK::needsTable)
    for (int i = lane; i < kNearExpTable; i += 32) tab[i] = A.expTable[i];
  __syncwarp();

  // Dynamic schedule (tile costs vary with leaf sizes: a static round-robin
  // measured 3-17% slower): tile k+2's index is claimed from the launch's
  // counter while tile k runs (the atomic's result is stored to shared memory
  // only after the tile's last chunk, so its latency is hidden), and tile
  // k+1's descriptor is loaded into registers when tile k starts, so the copy
  // issue never waits on memory. The first two tiles of each CTA are static.
  struct Next {
    FktbTile tile;
    int sb, se;
  };
  auto fetch = [&](int u) {
    Next x{};
    if (u < A.tile1) {
      x.tile = A.tiles[u / PARTS];
      x.sb = static_cast<int>(A.begin[x.tile.node]);
      x.se = static_cast<int>(A.end[x.tile.node]);
    }
    return x;
  };
  // issue the bulk copies of rows [s0, s0 + cnt) into stage st (one thread)
  auto issue = [&](int s0, int cnt, int st) {
    double* g = stage0 + st * SM::kStage;
    double* wv = g + SM::kGeo;
    const uint32_t gb = static_cast<uint32_t>(cnt) * GS * 8;
    const uint32_t wb = static_cast<uint32_t>(cnt) * RP * 8;
    mbar_expect_tx(bar + st, gb + wb);
    bulk_copy(g, A.rows + static_cast<size_t>(s0) * GS, gb, bar + st);
    if constexpr (RP > 0) bulk_copy(wv, A.w + static_cast<size_t>(s0) * RP, wb, bar + st);
  };

  __shared__ int sQ[3];  // tile indices, ring over k mod 3
  int t = A.tile0 + blockIdx.x;
  if (t >= A.tile1) return;
  if (lane == 0) sQ[1] = t + gridDim.x;
  Next cur = fetch(t);
  if (lane == 0) issue(cur.sb, min(CH, cur.se - cur.sb), 0);
  int st = 0, k = 0;
  uint32_t phase = 0;  // bit s: parity to wait for on stage s
  __syncwarp();

  while (t < A.tile1) {
    const int tn1 = sQ[(k + 1) % 3];
    const Next nxt = fetch(tn1);  // consumed at this tile's last chunk
    int claimed = 0;
    if (lane == 0) claimed = atomicAdd(A.counter, 1) + A.tile0 + 2 * static_cast<int>(gridDim.x);
    const FktbTile tile = cur.tile;
    const int leaf = tile.node;
    const int sb = cur.sb, se = cur.se;
    const int nch = (se - sb + CH - 1) / CH;
    const int base = (t % PARTS) * 32 * TPT;
    const bool active = base < tile.count;
    double c[D];
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = GRAM ? A.center[static_cast<size_t>(leaf) * D + a] : 0.0;
    const double Bt = FAC ? fma(1.000001 * kGramBound / A.gramLimit2, A.limit2[leaf], 1e-30) : 0.0;
    int tpos[TPT];
    double tx[TPT][D], tn[TPT], acc[TPT][R];
#pragma unroll
    for (int i = 0; i < TPT; ++i) {
      const int idx = base + lane + i * 32;
      tpos[i] = idx < tile.count ? static_cast<int>(A.nearPos[tile.start + idx]) : -1;
      const int p = tpos[i] >= 0 ? tpos[i] : 0;
      tn[i] = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        tx[i][a] = __dmul_rn(A.pc[static_cast<size_t>(a) * n + p] - c[a], A.sc);
        if constexpr (GRAM) tn[i] = fma(tx[i][a], tx[i][a] * (FAC ? 1.0 : FK::gramScale), tn[i]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
    }
    // Coincident (r == 0) pairs only occur inside a leaf: every split sends
    // equal coordinates to the same child (tree.cpp:93-171), so two points at
    // the same position share their leaf. Only the parts that hold targets of
    // the source leaf itself pay for the select (inverse-r at cfg4: 1 of ~25
    // near leaves per target).
    bool selPart = false;
    if constexpr (SEL) {
      bool mine = false;
#pragma unroll
      for (int i = 0; i < TPT; ++i) mine |= tpos[i] >= sb && tpos[i] < se;
      selPart = __any_sync(0xffffffffu, mine);
    }
    for (int ci = 0; ci < nch; ++ci) {
      if (lane == 0) {
        if (ci + 1 < nch)
          issue(sb + (ci + 1) * CH, min(CH, se - sb - (ci + 1) * CH), st ^ 1);
        else if (tn1 < A.tile1)
          issue(nxt.sb, min(CH, nxt.se - nxt.sb), st ^ 1);
      }
      const int s0 = sb + ci * CH;
      const int cn = min(CH, se - s0);
      const double* g = stage0 + st * SM::kStage;
      const double* wv = g + SM::kGeo;
      mbar_wait(bar + st, (phase >> st) & 1u);
      phase ^= 1u << st;
      // the chunk against this lane's TPT targets, with (selTag true) or
      // without the explicit r == 0 select
      auto evalChunk = [&](auto selTag) {
        constexpr bool kSel = decltype(selTag)::value;
        // the pair block of one source row against this lane's TPT targets
        auto pairs = [&](const double(&src)[GS], const double(&wr)[R]) {
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
            double kv = FK::template eval<1, GRAM>(q, tab, 0);
            // r == 0 <=> q == kQBias; compared on the high word (integer pipe):
            // any other q is >= ~1e-284 (points closer than ~1e-142 count as
            // coincident, where the FP64 form was already off)
            if constexpr (kSel) kv = __double2hiint(q) == kQBiasHi ? A.diagCanon : kv;
#pragma unroll
            for (int r = 0; r < R; ++r) acc[i][r] = fma(kv, wr[r], acc[i][r]);
          }
        };
        auto load = [&](double(&src)[GS], double(&wr)[R], int s) {
#pragma unroll
          for (int q = 0; q < GS; q += 2) {
            const double2 v = *reinterpret_cast<const double2*>(&g[s * GS + q]);
            src[q] = v.x;
            src[q + 1] = v.y;
          }
          if constexpr (RP == 0) {
            wr[0] = src[GS - 1];
          } else {
#pragma unroll
            for (int r = 0; r < R; r += 2) {
              const double2 v = *reinterpret_cast<const double2*>(&wv[s * RP + r]);
              wr[r] = v.x;
              if (r + 1 < R) wr[r + 1] = v.y;
            }
          }
        };
        if constexpr (nearPrefetch(D, R)) {
          // software pipeline: row s + 1 is loaded while row s is evaluated;
          // row cn is the stage's padding row (loaded, never used)
          double cur[GS], cw[R];
          load(cur, cw, 0);
#pragma unroll kNearUnroll
          for (int s = 0; s < cn; ++s) {
            double nx[GS], nw[R];
            load(nx, nw, s + 1);
            pairs(cur, cw);
#pragma unroll
            for (int q = 0; q < GS; ++q) cur[q] = nx[q];
#pragma unroll
            for (int r = 0; r < R; ++r) cw[r] = nw[r];
          }
        } else {
#pragma unroll kNearUnroll
          for (int s = 0; s < cn; ++s) {
            double src[GS], wr[R];
            load(src, wr, s);
            pairs(src, wr);
          }
        }
      };
      if (active) {
        if constexpr (SEL) {
          if (selPart)
            evalChunk(std::true_type{});
          else
            evalChunk(std::false_type{});
        } else {
          evalChunk(std::false_type{});
        }
      }
      if (lane == 0 && ci + 1 == nch) sQ[(k + 2) % 3] = claimed;
      __syncwarp();  // stage st is free for the copy issued next iteration
      st ^= 1;
    }
    if (active) {
#pragma unroll
      for (int i = 0; i < TPT; ++i)
        if (tpos[i] >= 0) {
          const double f = FAC ? A.scale * exp(-tn[i]) : A.scale;  // factored Gaussian: e^-|t|^2
#pragma unroll
          for (int r = 0; r < R; ++r) A.out.add(r, tile.start + base + lane + i * 32, tpos[i], acc[i][r] * f);
        }
    }
    t = tn1;
    cur = nxt;
    ++k;
  }
}

// Near-field configuration of a plan (fast path): scales, forms, rows.
struct NearFast {
  double sc = 1.0, wf = 1.0, diagCanon = 0.0, gramLimit2 = -1.0;
  bool sel = false;
};

template <int KID>
NearFast nearFastConfig(const DevicePlan& plan) {
  const DeviceTree& t = *plan.tree;
  FktbKernelDesc kd;
  fillKernelDesc(plan.kernel, kd);
  if (plan.options.hasDiagonal) kd.diag = plan.options.diagonal;
  NearFast f;
  fastScales(kd, f.sc, f.wf);
  f.diagCanon = kd.diag / f.wf;
  // The canonical formula already gives the reference convention at r == 0
  // for the smooth kernels (K(0) = valueAtZero); otherwise select explicitly.
  const bool smooth = KID != FKTB_KERNEL_INVERSE_R && KID != FKTB_KERNEL_INVERSE_R2;
  f.sel = !(smooth && kd.diag == f.wf);
  // Gram tiles only without the select (it needs exact r == 0 detection);
  // gramLimit2 < 0 leaves every tile to the difference form.
  if (FastKernel<KID>::gram && !f.sel)
    f.gramLimit2 = kGramBound / (f.sc * f.sc * (1.0 + t.theta * t.theta));
  return f;
}

template <int KID, int D, bool SEL, int TPT, int R, bool GRAM>
void launchStream(const DevicePlan& plan, const NearFast& f, const double* w, const ZOut& out, int tile0, int tile1,
                  int* counter, cudaStream_t st) {
  if (tile1 <= tile0) return;
  using FK = FastKernel<KID>;
  constexpr int GS = nearRowStride<KID>(D), RP = nearWStride(R);
  using SM = NearSmem<GS, RP, nearChunk(GS, RP), FK::needsTable>;
  auto kern = near_stream<KID, D, SEL, TPT, R, GRAM>;
  static int grid = 0;
  if (grid == 0) {
    FKTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SM::bytes)));
    int per = 0, dev = 0, sms = 148;
    FKTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32, SM::bytes));
    FKTB_CUDA(cudaGetDevice(&dev));
    FKTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, per) * sms;
  }
  const DeviceTree& t = *plan.tree;
  StreamArgs A{};
  A.n = t.n;
  A.pc = t.pc.get();
  A.begin = t.dBegin.get();
  A.end = t.dEnd.get();
  A.tiles = plan.dNearTiles.get();
  constexpr int PARTS = kNearTileTargets / (32 * TPT);
  A.tile0 = tile0 * PARTS;  // work units (tile, part)
  A.tile1 = tile1 * PARTS;
  A.nearPos = t.dNearPos.get();
  A.rows = plan.dNearRows.get();
  A.w = w;
  A.out = out;
  A.center = t.dCenter.get();
  A.limit2 = t.dLimit2.get();
  A.sc = f.sc;
  A.scale = GRAM && !FK::gramFactored ? f.wf * FK::gramWeight : f.wf;
  A.diagCanon = f.diagCanon;
  A.gramLimit2 = f.gramLimit2;
  A.expTable = expTableDevice(kNearExpBits, true);
  A.counter = counter;
  kern<<<std::min(grid, A.tile1 - A.tile0), 32, SM::bytes, st>>>(A);
  FKTB_CUDA(cudaGetLastError());
}

// One RHS pass of R columns: both pair forms (Gram tiles first).
template <int KID, int D, bool SEL, int TPT, int R>
void launchForms(const DevicePlan& plan, const NearFast& f, const double* w, const ZOut& out, cudaStream_t st) {
  const int tiles = static_cast<int>(plan.nearTilesHost.size()), g = plan.nearGramTileCount;
  FKTB_CUDA(cudaMemsetAsync(plan.dNearCounter.get(), 0, 2 * sizeof(int), st));
  if constexpr (FastKernel<KID>::gram && !SEL)
    launchStream<KID, D, SEL, TPT, R, true>(plan, f, w, out, 0, g, plan.dNearCounter.get(), st);
  launchStream<KID, D, SEL, TPT, R, false>(plan, f, w, out, g, tiles, plan.dNearCounter.get() + 1, st);
}

template <int KID, int D, bool SEL, int TPT, int R>
void launchPasses(const DevicePlan& plan, const NearFast& f, const double* yp, const ZOut& out, int nrhs, cudaStream_t st) {
  const size_t n = static_cast<size_t>(plan.n);
  const bool fac = plan.dNearFac.get() != nullptr;
  for (int r0 = 0; r0 + R <= nrhs; r0 += R) {
    const double* y = yp + r0 * n;
    const double* w = nullptr;
    const int blocks = static_cast<int>((n + 255) / 256);
    if constexpr (R == 1) {
      near_fill_weights<<<blocks, 256, 0, st>>>(y, fac ? plan.dNearFac.get() : nullptr, plan.dNearRows.get(), plan.n,
                                                nearRowStride<KID>(D));
    } else {
      near_weights_kernel<<<blocks, 256, 0, st>>>(y, fac ? plan.dNearFac.get() : nullptr, plan.dNearW.get(), plan.n, R,
                                                  nearWStride(R));
      w = plan.dNearW.get();
    }
    FKTB_CUDA(cudaGetLastError());
    launchForms<KID, D, SEL, TPT, R>(plan, f, w, zoutShift(out, r0), st);
  }
}

template <int KID, int D, bool SEL>
void launchFastSel(const DevicePlan& plan, const NearFast& f, const double* yp, const ZOut& zp, int nrhs, cudaStream_t st) {
  // targets per lane (measured shapes, B200 sweeps): Matern-3/2 in 3-D 8
  // independent targets; the others 4; 16 RHS: 4 targets x 16 accumulators
  // (each source's 16 weights serve 64 FMAs); 4/8 RHS: 2 targets
  if (nrhs % 16 == 0) return launchPasses<KID, D, SEL, 4, 16>(plan, f, yp, zp, nrhs, st);
  if (nrhs % 8 == 0) return launchPasses<KID, D, SEL, 2, 8>(plan, f, yp, zp, nrhs, st);
  if (nrhs % 4 == 0) return launchPasses<KID, D, SEL, 2, 4>(plan, f, yp, zp, nrhs, st);
  if (nrhs % 2 == 0) return launchPasses<KID, D, SEL, 4, 2>(plan, f, yp, zp, nrhs, st);
  if constexpr (KID == FKTB_KERNEL_MATERN32 && D == 3 && !SEL) return launchPasses<KID, D, SEL, 8, 1>(plan, f, yp, zp, nrhs, st);
  if constexpr (KID == FKTB_KERNEL_GAUSSIAN && D == 5 && !SEL && FKTB_NEAR_G5_TPT == 8)
    return launchPasses<KID, D, SEL, 8, 1>(plan, f, yp, zp, nrhs, st);
  return launchPasses<KID, D, SEL, 4, 1>(plan, f, yp, zp, nrhs, st);
}

template <int KID, int D>
void launchFastT(const DevicePlan& plan, const double* yp, const ZOut& zp, int nrhs, cudaStream_t st) {
  const NearFast f = nearFastConfig<KID>(plan);
  if (f.sel)
    launchFastSel<KID, D, true>(plan, f, yp, zp, nrhs, st);
  else
    launchFastSel<KID, D, false>(plan, f, yp, zp, nrhs, st);
}

// Plan time: Gram-first tile order, per-leaf forms, geometry rows.
template <int KID, int D>
void buildRowsT(DevicePlan& plan) {
  using FK = FastKernel<KID>;
  const DeviceTree& t = *plan.tree;
  const NearFast f = nearFastConfig<KID>(plan);
  std::vector<unsigned char> leafGram(static_cast<size_t>(t.nodes), 0);
  if (f.gramLimit2 >= 0.0)
    for (int b = 0; b < t.nodes; ++b) {
      volatile double limit = t.radius[static_cast<size_t>(b)] / t.theta;  // as tree.cu's limit2
      leafGram[static_cast<size_t>(b)] = limit * limit <= f.gramLimit2;
    }
  std::stable_partition(plan.nearTilesHost.begin(), plan.nearTilesHost.end(),
                        [&](const FktbTile& tl) { return leafGram[static_cast<size_t>(tl.node)] != 0; });
  plan.nearGramTileCount = 0;
  for (const FktbTile& tl : plan.nearTilesHost) plan.nearGramTileCount += leafGram[static_cast<size_t>(tl.node)];
  if (plan.nearRowsBuilt) return;  // rows depend on the tree and kernel only (not on the shard)
  constexpr int GS = nearRowStride<KID>(D);
  const size_t n = static_cast<size_t>(t.n);
  plan.dNearRows.resize(n * GS + GS);
  if (FK::gramFactored && f.gramLimit2 >= 0.0) plan.dNearFac.resize(n + 2);
  DeviceBuffer<unsigned char> dLeafGram(leafGram.size());
  FKTB_CUDA(cudaMemcpyAsync(dLeafGram.get(), leafGram.data(), leafGram.size(), cudaMemcpyHostToDevice, plan.stream));
  RowArgs A{t.n, t.pc.get(), t.dBegin.get(), t.dEnd.get(), t.dLeft.get(), t.dCenter.get(), t.dLimit2.get(),
            dLeafGram.get(), f.sc, f.gramLimit2, plan.dNearRows.get(), plan.dNearFac.get()};
  near_rows_kernel<KID, D><<<t.nodes, 128, 0, plan.stream>>>(A);
  FKTB_CUDA(cudaGetLastError());
  FKTB_CUDA(cudaStreamSynchronize(plan.stream));  // dLeafGram is a temporary
  plan.nearRowsBuilt = true;
}

template <int KID>
bool buildRowsK(DevicePlan& plan) {
  if constexpr (FastKernel<KID>::supported) {
    switch (plan.d) {
      case 2: buildRowsT<KID, 2>(plan); return true;
      case 3: buildRowsT<KID, 3>(plan); return true;
      case 5: buildRowsT<KID, 5>(plan); return true;
      default: break;
    }
  }
  return false;
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
    if (plan.nearRowsBuilt) switch (A.d) {
      case 2: return launchFastT<KID, 2>(plan, A.yp, A.out, A.nrhs, st);
      case 3: return launchFastT<KID, 3>(plan, A.yp, A.out, A.nrhs, st);
      case 5: return launchFastT<KID, 5>(plan, A.yp, A.out, A.nrhs, st);
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
// per (size, form), built once (outside any graph capture: see createPlan).
// compensated: the high word of entry j is lowered by j << (20 - bits), the
// form exp_neg_fi reads (its exponent step adds it back with kb's low bits).
const double* expTableDevice(int bits, bool compensated) {
  static double* dev[2][16] = {};
  static std::once_flag once[2][16];
  if (bits < 0 || bits >= 16 || (compensated && bits > 20)) throw std::invalid_argument("exp table size");
  const int c = compensated ? 1 : 0;
  std::call_once(once[c][bits], [bits, c] {
    const int n = 1 << bits;
    std::vector<double> host(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) {
      double v = static_cast<double>(std::exp2(static_cast<long double>(j) / n));
      if (c) {
        uint64_t u;
        std::memcpy(&u, &v, sizeof u);
        const uint32_t hi = static_cast<uint32_t>(u >> 32) - (static_cast<uint32_t>(j) << (20 - bits));
        u = (static_cast<uint64_t>(hi) << 32) | (u & 0xffffffffull);
        std::memcpy(&v, &u, sizeof v);
      }
      host[static_cast<size_t>(j)] = v;
    }
    FKTB_CUDA(cudaMalloc(&dev[c][bits], host.size() * sizeof(double)));
    FKTB_CUDA(cudaMemcpy(dev[c][bits], host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice));
  });
  return dev[c][bits];
}

int nearTileSize() { return kNearTileTargets; }

// Gram-form tiles of the FP64 fast near field (0 when the plan's kernel,
// dimension or diagonal convention keeps the difference form).
long long nearGramTiles(const DevicePlan& plan) { return plan.nearRowsBuilt ? plan.nearGramTileCount : 0; }

// True when the plan runs the streaming fast path (near_stream).
bool nearFastPath(const DevicePlan& plan) { return plan.nearRowsBuilt; }

// Plan time (and after every re-tiling): tile order, per-leaf forms and, once,
// the geometry rows of the fast path.
void buildNearRows(DevicePlan& plan) {
  switch (plan.kernel.id) {
    case FKTB_KERNEL_EXPONENTIAL: buildRowsK<FKTB_KERNEL_EXPONENTIAL>(plan); return;
    case FKTB_KERNEL_MATERN12: buildRowsK<FKTB_KERNEL_MATERN12>(plan); return;
    case FKTB_KERNEL_MATERN32: buildRowsK<FKTB_KERNEL_MATERN32>(plan); return;
    case FKTB_KERNEL_CAUCHY: buildRowsK<FKTB_KERNEL_CAUCHY>(plan); return;
    case FKTB_KERNEL_RATIONAL_QUADRATIC: buildRowsK<FKTB_KERNEL_RATIONAL_QUADRATIC>(plan); return;
    case FKTB_KERNEL_GAUSSIAN: buildRowsK<FKTB_KERNEL_GAUSSIAN>(plan); return;
    case FKTB_KERNEL_INVERSE_R: buildRowsK<FKTB_KERNEL_INVERSE_R>(plan); return;
    case FKTB_KERNEL_INVERSE_R2: buildRowsK<FKTB_KERNEL_INVERSE_R2>(plan); return;
    default: return;
  }
}


// Near-field launches of one multiply (kernelLaunches).
long long nearLaunches(const DevicePlan& plan, int nrhs) {
  if (plan.nearTilesHost.empty()) return 0;
  if (!plan.nearRowsBuilt) return 1;  // generic kernel: every RHS in one launch
  const int r = nrhs % 16 == 0 ? 16 : nrhs % 8 == 0 ? 8 : nrhs % 4 == 0 ? 4 : nrhs % 2 == 0 ? 2 : 1;
  const long long g = plan.nearGramTileCount, t = static_cast<long long>(plan.nearTilesHost.size());
  const long long perPass = (g > 0) + (g < t) + 1;  // + the weight kernel
  return perPass * (nrhs / r);
}

void launchNear(const DevicePlan& plan, const double* yp, double* zp, int nrhs, cudaStream_t st) {
  const int tiles = static_cast<int>(plan.nearTilesHost.size());
  if (tiles == 0) return;
  const DeviceTree& t = *plan.tree;
  NearArgs A{t.n, t.d, nrhs, t.pc.get(), t.dBegin.get(), t.dEnd.get(), plan.dNearTiles.get(), t.dNearPos.get(), yp,
             zoutFor(plan, zp, nrhs, false), {}};
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
