// K4 (source-to-multipole) and K5 (multipole-to-target) far field.
//
// Reference: proj/src/transform.cpp:131-161 (streaming path), operator rows /
// columns from proj/src/expansion.cpp:263-355, radial coefficients
// expansion.cpp:12-44, harmonics harmonics.cpp:160-246.
//
//   M_b[k,h,s] = Z_k nrm_h^2 * sum_{src in b} Yraw_h(x'_src) R_{k,s}(r'_src) y_src
//   z_t      += sum_{k,s} W_{k,s}(r_t) sum_h Yraw_h(x_t) M_b[k,h,s]   (t in F_b)
// where uncompressed R_{k,s}(r') = r'^(k+2s) and
//   W_{k,s}(r) = r^-j sum_{m=1..j} (K^(m)(r)/m!) r^m (Tbar_kjm m!)  (+K(r) at k=j=0),
// compressed R = G_{k,i}(r'), W = K(r) F_{k,i}(r). The normalisers of the
// reference's orthonormal basis (nrm_h) and addition theorem (Z_k) are folded
// into the moments, so the per-pair work only evaluates raw chain products.
//
// K4: CTA per (node, source tile); per-coefficient warp reductions into
// per-warp shared slots; one global atomic per coefficient per tile.
// K5: CTA per (node, <=128 far targets); node moments staged in shared
// memory (broadcast reads); thread per target evaluates harmonics, kernel jet
// and radial table (kernel-parameter constant bank) and contracts.
#include "device_math.cuh"
#include "plan.hpp"

namespace fktb {
namespace {

constexpr int kS2MThreads = 128;
constexpr int kM2TThreads = 128;
constexpr int kGenericGMax = 546;  // (d-2)(p+1)(p+2)/2 bound for the runtime path

struct FarArgs {
  int n;
  int nrhs;
  const double* pc;
  const double* center;
  const FktbTile* tiles;
  const uint32_t* farPos;
  const double* hscale;
  const int* chainG;
  const int* chainC;
  const int* chainPh;
  const double* yp;
  double* zp;
  double* moments;
};

// Uncompressed radial slot value R_{k,s}(r') or compressed source factor.
template <int P>
__device__ __forceinline__ double poly_eval(const FktbFarParams& fp, int f, double x) {
  // sum_{e=gLo..gHi} c_e x^e, Horner from the top, times x^gLo.
  const int lo = fp.gLo[f], hi = fp.gHi[f], at = fp.gAt[f];
  double acc = 0.0;
  for (int e = hi; e >= lo; --e) acc = fma(acc, x, fp.fc[at + e - lo]);
  double xp = 1.0;
  for (int e = 0; e < lo; ++e) xp *= x;
  return acc * xp;
}

__device__ __forceinline__ double laurent_eval(const FktbFarParams& fp, int f, double r, double rinv) {
  const int lo = fp.fLo[f], hi = fp.fHi[f], at = fp.fAt[f];
  double acc = 0.0;
  for (int e = hi; e >= lo; --e) acc = fma(acc, r, fp.fc[at + e - lo]);
  // times r^lo (lo may be negative)
  double sc = 1.0;
  if (lo >= 0)
    for (int e = 0; e < lo; ++e) sc *= r;
  else
    for (int e = 0; e < -lo; ++e) sc *= rinv;
  return acc * sc;
}

// Radial weights W_{k,s}(r) for all (k, s) into w[] (coefficient-slot order
// cOff-independent: index tOff[k] + s). Uncompressed path.
template <int PT>
__device__ __forceinline__ void radial_uncompressed(const FktbFarParams& fp, double r, double* w) {
  constexpr int NP = PT > 0 ? PT : FKTB_MAX_P;
  const int p = PT > 0 ? PT : fp.p;
  Jet<NP> c;
  kernel_jet<NP>(fp.kernel, r, c, p);
  const double rinv = 1.0 / r;
  double q[NP + 1];  // q_m = c_m r^m
  {
    double rm = 1.0;
#pragma unroll
    for (int m = 0; m <= NP; ++m) {
      if (m > p) break;
      q[m] = c.c[m] * rm;
      rm *= r;
    }
  }
#pragma unroll
  for (int k = 0; k <= NP; ++k) {
    if (k > p) break;
    double rj = 1.0;  // r^-j, j = k + 2s
#pragma unroll
    for (int i = 0; i < k; ++i) rj *= rinv;
#pragma unroll
    for (int s = 0; 2 * s <= NP - k; ++s) {
      const int j = k + 2 * s;
      if (j > p) break;
      const int widx = PT > 0 ? slot_base(PT, k) + s : fp.tOff[k] + s;
      const int row = fp.tRow[widx];
      double acc = 0.0;
#pragma unroll
      for (int m = 1; m <= j; ++m) acc = fma(q[m], fp.tb[row + m - 1], acc);
      acc *= rj;
      if (j == 0) acc += c.c[0];
      w[widx] = acc;
      rj *= rinv * rinv;
    }
  }
}

// ----------------------------------------------------------------------------
// K4: source-to-multipole. Compile-time (D, P) or runtime (0, 0).
template <int D, int P>
__global__ void __launch_bounds__(kS2MThreads) s2m_kernel(const __grid_constant__ FktbFarParams fp,
                                                           const __grid_constant__ FarArgs A) {
  extern __shared__ double slots[];  // [warps][nrhs][P]
  const int d = D > 0 ? D : fp.d;
  const int p = P > 0 ? P : fp.p;
  const int PC = fp.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kS2MThreads / 32;
  const FktbTile tile = A.tiles[blockIdx.x];
  const int b = tile.node;
  for (int i = threadIdx.x; i < NW * PC * A.nrhs; i += kS2MThreads) slots[i] = 0.0;
  __syncthreads();
  constexpr int DD = D > 0 ? D : FKTB_MAX_DIM;
  double c[DD];
#pragma unroll
  for (int a = 0; a < DD; ++a)
    if (a < d) c[a] = A.center[static_cast<size_t>(b) * d + a];
  const int rounds = (tile.count + 31) / 32;
  for (int rd = warp; rd < rounds; rd += NW) {
    const int i = rd * 32 + lane;
    const bool valid = i < tile.count;
    const int pos = static_cast<int>(tile.start) + (valid ? i : 0);
    double x[DD];
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < DD; ++a)
      if (a < d) {
        x[a] = A.pc[static_cast<size_t>(a) * A.n + pos] - c[a];
        r2 = fma(x[a], x[a], r2);
      }
    const double r = sqrt(r2);
    if constexpr (D > 0) {
      constexpr int H = ChainTable<D, P>::H;
      double Y[H];
      harmonics_raw<D, P>(x, r, Y);
      // radial source values R_{k,s}(r')
      double rp[P + 1];
      rp[0] = 1.0;
#pragma unroll
      for (int m = 1; m <= P; ++m) rp[m] = rp[m - 1] * r;
      for (int rhs = 0; rhs < A.nrhs; ++rhs) {
        const double wgt = valid ? A.yp[static_cast<size_t>(rhs) * A.n + pos] : 0.0;
        double* sl = slots + (static_cast<size_t>(warp) * A.nrhs + rhs) * PC;
#pragma unroll
        for (int k = 0; k <= P; ++k) {
          const int ns = fp.slots[k];
#pragma unroll
          for (int h = harmonic_offset(D, k); h < harmonic_offset(D, k + 1); ++h) {
            const double yw = Y[h] * wgt;
#pragma unroll
            for (int s = 0; s < slots_u(P, k); ++s) {
              if (s >= ns) break;
              const double rv = fp.compressed ? poly_eval<P>(fp, fp.fOff[k] + s, r) : rp[k + 2 * s];
              const double v = warp_sum(yw * rv);
              if (lane == 0) sl[coef_offset(D, P, k) + (h - harmonic_offset(D, k)) * slots_u(P, k) + s] += v;
            }
          }
        }
      }
    } else {
      // Runtime (d, p): Gegenbauer tables in local memory, chains from global.
      const double inv = r > 0.0 ? 1.0 / r : 0.0;
      double v[FKTB_MAX_DIM];
      for (int a = 0; a < d; ++a) v[a] = x[a] * inv;
      double cA[FKTB_MAX_P + 1], cB[FKTB_MAX_P + 1];
      cA[0] = 1.0;
      cB[0] = 0.0;
      for (int m = 1; m <= p; ++m) {
        cA[m] = cA[m - 1] * v[d - 2] - cB[m - 1] * v[d - 1];
        cB[m] = cB[m - 1] * v[d - 2] + cA[m - 1] * v[d - 1];
      }
      double g[kGenericGMax];
      if (d > 2) {
        double tail[FKTB_MAX_DIM];
        double accT = 0.0;
        for (int q = d - 1; q >= 0; --q) {
          accT += v[q] * v[q];
          tail[q] = accT;
        }
        for (int level = 1; level <= d - 2; ++level) {
          const double xx = v[level - 1], t2 = tail[level - 1];
          for (int m = 0; m <= p; ++m) {
            const int twoLam = d - 1 - level + 2 * m;
            double* row = g + g_index(p, level, m, 0);
            row[0] = 1.0;
            if (p - m >= 1) row[1] = twoLam * xx;
            for (int nn = 2; nn <= p - m; ++nn)
              row[nn] = ((2 * nn + twoLam - 2) * xx * row[nn - 1] - (nn + twoLam - 2) * t2 * row[nn - 2]) / nn;
          }
        }
      }
      const int L = d > 2 ? d - 2 : 0;
      for (int k = 0; k <= p; ++k) {
        const int ns = fp.slots[k];
        for (int h = fp.hOff[k]; h < fp.hOff[k + 1]; ++h) {
          double yv = A.chainPh[h] >= 0 ? cA[A.chainC[h]] : cB[A.chainC[h]];
          for (int l = 0; l < L; ++l) yv *= g[A.chainG[h * L + l]];
          const int base = fp.cOff[k] + (h - fp.hOff[k]) * fp.slotsU[k];
          for (int s = 0; s < ns; ++s) {
            double rv;
            if (fp.compressed) {
              rv = poly_eval<0>(fp, fp.fOff[k] + s, r);
            } else {
              rv = 1.0;
              for (int e = 0; e < k + 2 * s; ++e) rv *= r;
            }
            for (int rhs = 0; rhs < A.nrhs; ++rhs) {
              const double wgt = valid ? A.yp[static_cast<size_t>(rhs) * A.n + pos] : 0.0;
              const double val = warp_sum(yv * rv * wgt);
              if (lane == 0) slots[(static_cast<size_t>(warp) * A.nrhs + rhs) * PC + base + s] += val;
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // Fold the normalisers and publish: one atomic per coefficient per tile.
  for (int i = threadIdx.x; i < PC * A.nrhs; i += kS2MThreads) {
    const int rhs = i / PC, cidx = i % PC;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) sum += slots[(static_cast<size_t>(w) * A.nrhs + rhs) * PC + cidx];
    // harmonic of coefficient cidx
    int k = 0;
    while (k < p && cidx >= fp.cOff[k + 1]) ++k;
    const int h = fp.hOff[k] + (cidx - fp.cOff[k]) / fp.slotsU[k];
    if ((cidx - fp.cOff[k]) % fp.slotsU[k] >= fp.slots[k]) continue;
    atomicAdd(A.moments + (static_cast<size_t>(b) * A.nrhs + rhs) * PC + cidx, sum * A.hscale[h]);
  }
}

// ----------------------------------------------------------------------------
// K5: multipole-to-target.
template <int D, int P>
__global__ void __launch_bounds__(kM2TThreads) m2t_kernel(const __grid_constant__ FktbFarParams fp,
                                                           const __grid_constant__ FarArgs A) {
  extern __shared__ double sM[];  // [nrhs][P]
  const int d = D > 0 ? D : fp.d;
  const int p = P > 0 ? P : fp.p;
  const int PC = fp.P;
  const FktbTile tile = A.tiles[blockIdx.x];
  const int b = tile.node;
  for (int i = threadIdx.x; i < PC * A.nrhs; i += kM2TThreads)
    sM[i] = A.moments[static_cast<size_t>(b) * A.nrhs * PC + i];
  __syncthreads();
  const int i = threadIdx.x;
  if (i >= tile.count) return;
  const int pos = static_cast<int>(A.farPos[tile.start + i]);
  constexpr int DD = D > 0 ? D : FKTB_MAX_DIM;
  double x[DD];
  double r2 = 0.0;
#pragma unroll
  for (int a = 0; a < DD; ++a)
    if (a < d) {
      x[a] = A.pc[static_cast<size_t>(a) * A.n + pos] - A.center[static_cast<size_t>(b) * d + a];
      r2 = fma(x[a], x[a], r2);
    }
  const double r = sqrt(r2);
  const double rinv = 1.0 / r;
  // Radial weights per (k, s).
  constexpr int WN = P > 0 ? (P / 2 + 1) * (P + 1) : (FKTB_MAX_P / 2 + 1) * (FKTB_MAX_P + 1);
  double w[WN];
  if (fp.compressed) {
    const double kv = kernel_value_rt(fp.kernel, r);
#pragma unroll
    for (int k = 0; k <= (P > 0 ? P : FKTB_MAX_P); ++k) {
      if (k > p) break;
      for (int s = 0; s < (P > 0 ? slots_u(P, k) : fp.slotsU[k]); ++s) {
        if (s >= fp.slots[k]) break;
        const int widx = P > 0 ? slot_base(P, k) + s : fp.tOff[k] + s;
        w[widx] = kv * laurent_eval(fp, fp.fOff[k] + s, r, rinv);
      }
    }
  } else {
    radial_uncompressed<P>(fp, r, w);
  }
  if constexpr (D > 0) {
    constexpr int H = ChainTable<D, P>::H;
    double Y[H];
    harmonics_raw<D, P>(x, r, Y);
    for (int rhs = 0; rhs < A.nrhs; ++rhs) {
      const double* M = sM + rhs * PC;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        const int ns = fp.slots[k];
#pragma unroll
        for (int s = 0; s < slots_u(P, k); ++s) {
          if (s >= ns) break;
          double inner = 0.0;
#pragma unroll
          for (int h = harmonic_offset(D, k); h < harmonic_offset(D, k + 1); ++h)
            inner = fma(Y[h], M[coef_offset(D, P, k) + (h - harmonic_offset(D, k)) * slots_u(P, k) + s], inner);
          acc = fma(w[slot_base(P, k) + s], inner, acc);
        }
      }
      atomicAdd(A.zp + static_cast<size_t>(rhs) * A.n + pos, acc);
    }
  } else {
    const double inv = rinv;
    double v[FKTB_MAX_DIM];
    for (int a = 0; a < d; ++a) v[a] = x[a] * inv;
    double cA[FKTB_MAX_P + 1], cB[FKTB_MAX_P + 1];
    cA[0] = 1.0;
    cB[0] = 0.0;
    for (int m = 1; m <= p; ++m) {
      cA[m] = cA[m - 1] * v[d - 2] - cB[m - 1] * v[d - 1];
      cB[m] = cB[m - 1] * v[d - 2] + cA[m - 1] * v[d - 1];
    }
    double g[kGenericGMax];
    if (d > 2) {
      double tail[FKTB_MAX_DIM];
      double accT = 0.0;
      for (int q = d - 1; q >= 0; --q) {
        accT += v[q] * v[q];
        tail[q] = accT;
      }
      for (int level = 1; level <= d - 2; ++level) {
        const double xx = v[level - 1], t2 = tail[level - 1];
        for (int m = 0; m <= p; ++m) {
          const int twoLam = d - 1 - level + 2 * m;
          double* row = g + g_index(p, level, m, 0);
          row[0] = 1.0;
          if (p - m >= 1) row[1] = twoLam * xx;
          for (int nn = 2; nn <= p - m; ++nn)
            row[nn] = ((2 * nn + twoLam - 2) * xx * row[nn - 1] - (nn + twoLam - 2) * t2 * row[nn - 2]) / nn;
        }
      }
    }
    const int L = d > 2 ? d - 2 : 0;
    for (int rhs = 0; rhs < A.nrhs; ++rhs) {
      const double* M = sM + rhs * PC;
      double acc = 0.0;
      for (int k = 0; k <= p; ++k) {
        const int ns = fp.slots[k];
        for (int h = fp.hOff[k]; h < fp.hOff[k + 1]; ++h) {
          double yv = A.chainPh[h] >= 0 ? cA[A.chainC[h]] : cB[A.chainC[h]];
          for (int l = 0; l < L; ++l) yv *= g[A.chainG[h * L + l]];
          const int base = fp.cOff[k] + (h - fp.hOff[k]) * fp.slotsU[k];
          double inner = 0.0;
          for (int s = 0; s < ns; ++s) inner = fma(w[fp.tOff[k] + s], M[base + s], inner);
          acc = fma(yv, inner, acc);
        }
      }
      atomicAdd(A.zp + static_cast<size_t>(rhs) * A.n + pos, acc);
    }
  }
}

template <int D, int P>
void launchFarT(const FktbFarParams& fp, const FarArgs& A, int tiles, bool s2m, cudaStream_t st) {
  if (s2m) {
    const size_t smem = static_cast<size_t>(kS2MThreads / 32) * fp.P * A.nrhs * sizeof(double);
    if (smem > 48 * 1024)
      FKTB_CUDA(cudaFuncSetAttribute(s2m_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    s2m_kernel<D, P><<<tiles, kS2MThreads, smem, st>>>(fp, A);
  } else {
    const size_t smem = static_cast<size_t>(fp.P) * A.nrhs * sizeof(double);
    if (smem > 48 * 1024)
      FKTB_CUDA(cudaFuncSetAttribute(m2t_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    m2t_kernel<D, P><<<tiles, kM2TThreads, smem, st>>>(fp, A);
  }
  FKTB_CUDA(cudaGetLastError());
}

void launchFar(const DevicePlan& plan, const FarArgs& A, int tiles, bool s2m, cudaStream_t st) {
  if (tiles == 0) return;
  const FktbFarParams& fp = *plan.far;
  const int key = fp.d * 100 + fp.p;
  switch (key) {
    case 206: return launchFarT<2, 6>(fp, A, tiles, s2m, st);
    case 304: return launchFarT<3, 4>(fp, A, tiles, s2m, st);
    case 306: return launchFarT<3, 6>(fp, A, tiles, s2m, st);
    case 308: return launchFarT<3, 8>(fp, A, tiles, s2m, st);
    case 504: return launchFarT<5, 4>(fp, A, tiles, s2m, st);
    default: return launchFarT<0, 0>(fp, A, tiles, s2m, st);
  }
}

}  // namespace

int farTileSize() { return kM2TThreads; }
int genericGMax() { return kGenericGMax; }

void launchS2M(const DevicePlan& plan, const double* yp, double* moments, int nrhs, cudaStream_t st) {
  const DeviceTree& t = *plan.tree;
  FarArgs A{t.n, nrhs, t.pc.get(), t.dCenter.get(), plan.dS2mTiles.get(), nullptr, plan.dHScale.get(),
            plan.dChainG.get(), plan.dChainC.get(), plan.dChainPh.get(), yp, nullptr, moments};
  launchFar(plan, A, static_cast<int>(plan.s2mTilesHost.size()), true, st);
}

void launchM2T(const DevicePlan& plan, const double* moments, double* zp, int nrhs, cudaStream_t st) {
  const DeviceTree& t = *plan.tree;
  FarArgs A{t.n, nrhs, t.pc.get(), t.dCenter.get(), plan.dFarTiles.get(), t.dFarPos.get(), plan.dHScale.get(),
            plan.dChainG.get(), plan.dChainC.get(), plan.dChainPh.get(), nullptr, zp, const_cast<double*>(moments)};
  launchFar(plan, A, static_cast<int>(plan.farTilesHost.size()), false, st);
}

}  // namespace fktb
