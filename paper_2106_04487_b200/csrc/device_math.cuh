// Device math for the FKT kernels (sm_100a): isotropic kernel evaluation
// (near field, dense rows), Taylor jets of the kernels (far-field radial
// coefficients) and raw hyperspherical-harmonic chains (s2m / m2t).
//
// Reference map:
//  * kernel formulas      proj/src/kernels.cpp:37-156
//  * jet arithmetic       proj/include/fkt/jet.hpp:88-210
//  * harmonic chains      proj/src/harmonics.cpp:160-246 (normalisation
//                          constants are folded into the node moments on the
//                          host side, see far.cu)
#ifndef FKTB_DEVICE_MATH_CUH
#define FKTB_DEVICE_MATH_CUH

#include "cart_layout.hpp"
#include "fkt_device_types.h"

namespace fktb {

// ---------------------------------------------------------------------------
// K(r) for r > 0 given dist2 = r^2 (and r when the formula needs it). Where the
// reference formula only involves r^2 the square root is skipped; the value
// differs from reference bits by roundoff only.
template <int KID>
struct KernelNeedsR {
  static constexpr bool value = !(KID == FKTB_KERNEL_CAUCHY || KID == FKTB_KERNEL_RATIONAL_QUADRATIC ||
                                  KID == FKTB_KERNEL_GAUSSIAN || KID == FKTB_KERNEL_INVERSE_R ||
                                  KID == FKTB_KERNEL_INVERSE_R2 || KID == FKTB_KERNEL_EXP_NEG_INV_R2);
};

template <int KID>
__device__ __forceinline__ double kernel_value(const FktbKernelDesc& k, double dist2) {
  if constexpr (KID == FKTB_KERNEL_CAUCHY) {
    return 1.0 / fma(dist2, k.is2, 1.0);
  } else if constexpr (KID == FKTB_KERNEL_RATIONAL_QUADRATIC) {
    return rsqrt(fma(dist2, k.is2, 1.0));
  } else if constexpr (KID == FKTB_KERNEL_GAUSSIAN) {
    return exp(-dist2);
  } else if constexpr (KID == FKTB_KERNEL_INVERSE_R) {
    return rsqrt(dist2);
  } else if constexpr (KID == FKTB_KERNEL_INVERSE_R2) {
    return 1.0 / dist2;
  } else if constexpr (KID == FKTB_KERNEL_EXP_NEG_INV_R2) {
    return exp(-(1.0 / dist2));
  } else {
    const double r = sqrt(dist2);
    if constexpr (KID == FKTB_KERNEL_EXPONENTIAL) return exp(-r);
    if constexpr (KID == FKTB_KERNEL_MATERN12) return k.s2 * exp(-r / k.rho);
    if constexpr (KID == FKTB_KERNEL_MATERN32) {
      const double ar = k.a * r;
      return k.s2 * (1.0 + ar) * exp(-ar);
    }
    if constexpr (KID == FKTB_KERNEL_INVERSE_R3) return 1.0 / (r * dist2);
    if constexpr (KID == FKTB_KERNEL_EXP_OVER_R) return exp(-r) / r;
    if constexpr (KID == FKTB_KERNEL_R_EXP) return r * exp(-r);
    if constexpr (KID == FKTB_KERNEL_COS_OVER_R) return cos(r) / r;
    if constexpr (KID == FKTB_KERNEL_EXP_NEG_INV_R) return exp(-(1.0 / r));
    return 0.0;
  }
}

// Runtime-dispatched K(r), r > 0 (far-field compressed path).
__device__ __forceinline__ double kernel_value_rt(const FktbKernelDesc& k, double r) {
  const double r2 = r * r;
  switch (k.id) {
    case FKTB_KERNEL_EXPONENTIAL: return exp(-r);
    case FKTB_KERNEL_MATERN12: return k.s2 * exp(-r / k.rho);
    case FKTB_KERNEL_MATERN32: return k.s2 * (1.0 + k.a * r) * exp(-(k.a * r));
    case FKTB_KERNEL_CAUCHY: return 1.0 / (1.0 + r2 * k.is2);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return 1.0 / sqrt(1.0 + r2 * k.is2);
    case FKTB_KERNEL_GAUSSIAN: return exp(-r2);
    case FKTB_KERNEL_INVERSE_R: return 1.0 / r;
    case FKTB_KERNEL_INVERSE_R2: return 1.0 / r2;
    case FKTB_KERNEL_INVERSE_R3: return 1.0 / (r2 * r);
    case FKTB_KERNEL_EXP_OVER_R: return exp(-r) / r;
    case FKTB_KERNEL_R_EXP: return r * exp(-r);
    case FKTB_KERNEL_COS_OVER_R: return cos(r) / r;
    case FKTB_KERNEL_EXP_NEG_INV_R: return exp(-(1.0 / r));
    case FKTB_KERNEL_EXP_NEG_INV_R2: return exp(-(1.0 / r2));
  }
  return 0.0;
}

// ---------------------------------------------------------------------------
// Truncated Taylor series of order N (coefficient m = f^(m)(r)/m!). The
// recurrences restate proj/include/fkt/jet.hpp:110-190; with N a compile-time
// constant everything stays in registers. `n` is the runtime order (<= N).
template <int N>
struct Jet {
  double c[N + 1];
};

template <int N>
__device__ __forceinline__ void jet_mul(const Jet<N>& a, const Jet<N>& b, Jet<N>& r, int n) {
#pragma unroll
  for (int i = 0; i <= N; ++i) {
    if (i > n) break;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j <= i; ++j) acc = fma(a.c[j], b.c[i - j], acc);
    r.c[i] = acc;
  }
}

template <int N>
__device__ __forceinline__ void jet_div(const Jet<N>& a, const Jet<N>& b, Jet<N>& r, int n) {
  const double inv = 1.0 / b.c[0];
#pragma unroll
  for (int i = 0; i <= N; ++i) {
    if (i > n) break;
    double acc = a.c[i];
#pragma unroll
    for (int j = 1; j <= i; ++j) acc = fma(-b.c[j], r.c[i - j], acc);
    r.c[i] = acc * inv;
  }
}

template <int N>
__device__ __forceinline__ void jet_recip(const Jet<N>& b, Jet<N>& r, int n) {
  const double inv = 1.0 / b.c[0];
#pragma unroll
  for (int i = 0; i <= N; ++i) {
    if (i > n) break;
    double acc = i == 0 ? 1.0 : 0.0;
#pragma unroll
    for (int j = 1; j <= i; ++j) acc = fma(-b.c[j], r.c[i - j], acc);
    r.c[i] = acc * inv;
  }
}

template <int N>
__device__ __forceinline__ void jet_exp(const Jet<N>& f, Jet<N>& g, int n) {
  g.c[0] = exp(f.c[0]);
#pragma unroll
  for (int m = 1; m <= N; ++m) {
    if (m > n) break;
    double acc = 0.0;
#pragma unroll
    for (int k = 1; k <= m; ++k) acc = fma(static_cast<double>(k) * f.c[k], g.c[m - k], acc);
    g.c[m] = acc * (1.0 / m);
  }
}

template <int N>
__device__ __forceinline__ void jet_sqrt(const Jet<N>& f, Jet<N>& g, int n) {
  g.c[0] = sqrt(f.c[0]);
  const double inv2 = 0.5 / g.c[0];
#pragma unroll
  for (int m = 1; m <= N; ++m) {
    if (m > n) break;
    double acc = f.c[m];
#pragma unroll
    for (int k = 1; k < m; ++k) acc = fma(-g.c[k], g.c[m - k], acc);
    g.c[m] = acc * inv2;
  }
}

template <int N>
__device__ __forceinline__ void jet_cos(const Jet<N>& f, Jet<N>& cj, int n) {
  Jet<N> s;
  s.c[0] = sin(f.c[0]);
  cj.c[0] = cos(f.c[0]);
#pragma unroll
  for (int m = 1; m <= N; ++m) {
    if (m > n) break;
    double sa = 0.0, ca = 0.0;
#pragma unroll
    for (int k = 1; k <= m; ++k) {
      const double kf = k * f.c[k];
      sa = fma(kf, cj.c[m - k], sa);
      ca = fma(-kf, s.c[m - k], ca);
    }
    s.c[m] = sa * (1.0 / m);
    cj.c[m] = ca * (1.0 / m);
  }
}

template <int N>
__device__ __forceinline__ void jet_scale(Jet<N>& a, double s, int n) {
#pragma unroll
  for (int i = 0; i <= N; ++i)
    if (i <= n) a.c[i] *= s;
}

template <int N>
__device__ __forceinline__ void jet_var(double r, Jet<N>& v, int n) {
#pragma unroll
  for (int i = 0; i <= N; ++i) v.c[i] = 0.0;
  v.c[0] = r;
  if (n >= 1) v.c[1] = 1.0;
}

// Jet of the kernel at r > 0 up to order n (reference kernels.hpp:61-64 with
// the generic lambdas of kernels.cpp). Closed forms where they are short.
template <int N>
__device__ __forceinline__ void kernel_jet(const FktbKernelDesc& k, double r, Jet<N>& out, int n) {
  switch (k.id) {
    case FKTB_KERNEL_EXPONENTIAL:
    case FKTB_KERNEL_MATERN12: {
      // c_m = s (-1/l)^m e^{-r/l} / m!
      const double il = k.id == FKTB_KERNEL_EXPONENTIAL ? 1.0 : 1.0 / k.rho;
      const double s = k.id == FKTB_KERNEL_EXPONENTIAL ? 1.0 : k.s2;
      double t = s * exp(-r * il);
#pragma unroll
      for (int m = 0; m <= N; ++m) {
        out.c[m] = t;
        t *= -il / (m + 1);
      }
      return;
    }
    case FKTB_KERNEL_MATERN32: {
      // d^m/dr^m (1 + a r) e^{-a r} = (-a)^m (a r - m + 1) e^{-a r}
      const double ar = k.a * r;
      double t = k.s2 * exp(-ar);
#pragma unroll
      for (int m = 0; m <= N; ++m) {
        out.c[m] = t * (ar - m + 1.0);
        t *= -k.a / (m + 1);
      }
      return;
    }
    case FKTB_KERNEL_INVERSE_R: {
      // c_m = (-1)^m r^{-m-1}
      const double ir = 1.0 / r;
      double t = ir;
#pragma unroll
      for (int m = 0; m <= N; ++m) {
        out.c[m] = t;
        t *= -ir;
      }
      return;
    }
    default:
      break;
  }
  Jet<N> v, a, b;
  jet_var(r, v, n);
  switch (k.id) {
    case FKTB_KERNEL_CAUCHY:
    case FKTB_KERNEL_RATIONAL_QUADRATIC:
      jet_mul(v, v, a, n);
      jet_scale(a, k.is2, n);
      a.c[0] += 1.0;
      if (k.id == FKTB_KERNEL_CAUCHY) {
        jet_recip(a, out, n);
      } else {
        jet_sqrt(a, b, n);
        jet_recip(b, out, n);
      }
      return;
    case FKTB_KERNEL_GAUSSIAN:
      jet_mul(v, v, a, n);
      jet_scale(a, -1.0, n);
      jet_exp(a, out, n);
      return;
    case FKTB_KERNEL_INVERSE_R2:
      jet_mul(v, v, a, n);
      jet_recip(a, out, n);
      return;
    case FKTB_KERNEL_INVERSE_R3:
      jet_mul(v, v, a, n);
      jet_mul(a, v, b, n);
      jet_recip(b, out, n);
      return;
    case FKTB_KERNEL_EXP_OVER_R:
      jet_scale(v, -1.0, n);
      jet_exp(v, a, n);
      jet_var(r, v, n);
      jet_div(a, v, out, n);
      return;
    case FKTB_KERNEL_R_EXP:
      jet_scale(v, -1.0, n);
      jet_exp(v, a, n);
      jet_var(r, v, n);
      jet_mul(v, a, out, n);
      return;
    case FKTB_KERNEL_COS_OVER_R:
      jet_cos(v, a, n);
      jet_div(a, v, out, n);
      return;
    case FKTB_KERNEL_EXP_NEG_INV_R:
      jet_recip(v, a, n);
      jet_scale(a, -1.0, n);
      jet_exp(a, out, n);
      return;
    case FKTB_KERNEL_EXP_NEG_INV_R2:
      jet_mul(v, v, a, n);
      jet_recip(a, b, n);
      jet_scale(b, -1.0, n);
      jet_exp(b, out, n);
      return;
    default:
#pragma unroll
      for (int m = 0; m <= N; ++m) out.c[m] = 0.0;
      return;
  }
}

// ---------------------------------------------------------------------------
// Compile-time harmonic chain tables (same enumeration as
// proj/src/harmonics.cpp:62-103): for each harmonic, the Gegenbauer table
// entry per level, the circular index and the cos/sin phase.
constexpr int harmonic_count_deg(int d, int k) {
  // binom(k+d-1, k) - binom(k+d-3, k-2)
  auto binom = [](int n, int r) -> long long {
    if (r < 0 || n < 0 || r > n) return 0;
    long long b = 1;
    for (int i = 1; i <= r; ++i) b = b * (n - r + i) / i;
    return b;
  };
  return static_cast<int>(binom(k + d - 1, k) - binom(k + d - 3, k - 2));
}

constexpr int harmonic_count(int d, int p) {
  int h = 0;
  for (int k = 0; k <= p; ++k) h += harmonic_count_deg(d, k);
  return h;
}

// Exponent window of the compressed target factors F_ki(r) for the builtin
// recurrence kernels (derived from q in K' = q K, expansion.cpp:179-212):
// inverse powers and constant q give r^-j (j <= p); gaussian gives [-p, p].
constexpr int compressed_window_lo(int kid, int p) {
  return kid == FKTB_KERNEL_GAUSSIAN || kid == FKTB_KERNEL_INVERSE_R || kid == FKTB_KERNEL_INVERSE_R2 ||
                 kid == FKTB_KERNEL_INVERSE_R3 || kid == FKTB_KERNEL_EXPONENTIAL || kid == FKTB_KERNEL_MATERN12
             ? -p
             : -2 * p;
}
constexpr int compressed_window_hi(int kid, int p) {
  return kid == FKTB_KERNEL_INVERSE_R || kid == FKTB_KERNEL_INVERSE_R2 || kid == FKTB_KERNEL_INVERSE_R3 ||
                 kid == FKTB_KERNEL_EXPONENTIAL || kid == FKTB_KERNEL_MATERN12
             ? 0
             : p;
}

// Compressed M2T, per kernel id: slots actually used per degree (the exact
// rank of the radial compression, known per kernel family) and the per-degree
// Laurent window of the target factors F_{k,i}. Laplace 1/r: rank 1 and
// F_k ~ r^-k (the multipole series 1/|x-y| = sum_k r'^k / r^(k+1) P_k).
// The host (buildFarParams) verifies the plan's factors against these before
// the specialised kernel may run.
constexpr int comp_slots(int kid, int p, int k) {
  return kid == FKTB_KERNEL_INVERSE_R ? 1 : (p - k) / 2 + 1;
}
// Kernels whose compression rank equals comp_slots at every degree (verified
// per plan): the fused M2T then needs no per-slot select and its factor rows
// sit at compile-time offsets.
constexpr bool comp_rank_exact(int kid) { return kid == FKTB_KERNEL_INVERSE_R; }
constexpr int comp_slot_base(int kid, int p, int k) {
  int s = 0;
  for (int q = 0; q < k; ++q) s += comp_slots(kid, p, q);
  return s;
}
constexpr int comp_degree_lo(int kid, int p, int k) {
  return kid == FKTB_KERNEL_INVERSE_R ? -k : compressed_window_lo(kid, p);
}
constexpr int comp_degree_hi(int kid, int p, int k) {
  return kid == FKTB_KERNEL_INVERSE_R ? -k : compressed_window_hi(kid, p);
}

constexpr int harmonic_offset(int d, int k) {
  int h = 0;
  for (int q = 0; q < k; ++q) h += harmonic_count_deg(d, q);
  return h;
}
constexpr int slots_u(int p, int k) { return (p - k) / 2 + 1; }
// First m with a possibly nonzero T-bar_kjm: in d = 3 the entries with
// m <= j - k - 2 vanish exactly (10 of 62 at p = 6, 29 of 130 at p = 8;
// verified entry by entry when a plan is built, plan.cu buildFarParams), so
// the compiled d = 3 radial weights skip them.
constexpr int tbarFirstM(int d, int k, int j) { return d == 3 && j - k - 1 > 1 ? j - k - 1 : 1; }

constexpr int slot_base(int p, int k) {
  int s = 0;
  for (int q = 0; q < k; ++q) s += slots_u(p, q);
  return s;
}
constexpr int coef_offset(int d, int p, int k) {
  int c = 0;
  for (int q = 0; q < k; ++q) c += harmonic_count_deg(d, q) * slots_u(p, q);
  return c;
}

// Monic-scaled homogeneous Gegenbauer recurrence. The reference's
// t^n C_n^(lambda)(x/t) (harmonics.cpp:212-230) satisfies
//   g_n = a_n x g_{n-1} - b_n t^2 g_{n-2},  a_n = (2n+2lam-2)/n, b_n = (n+2lam-2)/n;
// with g_n = kappa_n gh_n, kappa_n = a_1 ... a_n, the scaled values obey
//   gh_n = x gh_{n-1} - beta_n t^2 gh_{n-2},  beta_n = b_n / (a_n a_{n-1}),
// one multiply fewer per entry. The per-harmonic product of the kappas is
// folded into the node moments on the host (plan.cu, moments.cpp).
constexpr double gegen_a(int twoLam, int n) { return static_cast<double>(2 * n + twoLam - 2) / n; }
constexpr double gegen_beta(int twoLam, int n) {
  return (static_cast<double>(n + twoLam - 2) / n) / (gegen_a(twoLam, n) * gegen_a(twoLam, n - 1));
}
constexpr double gegen_kappa(int twoLam, int n) {
  double k = 1.0;
  for (int i = 1; i <= n; ++i) k *= gegen_a(twoLam, i);
  return k;
}

// Per-level Gegenbauer table g[level][m][n], n <= P - m: flat offset.
constexpr int g_level_size(int P) { return (P + 1) * (P + 2) / 2; }
constexpr int g_index(int P, int level, int m, int n) {
  return (level - 1) * g_level_size(P) + (m * (2 * P + 3 - m)) / 2 + n;
}

template <int D, int P>
struct ChainTable {
  static constexpr int H = harmonic_count(D, P);
  static constexpr int L = D > 2 ? D - 2 : 1;
  int gi[H][L];
  int ci[H];
  int ph[H];
  int deg[H];
};

template <int D, int P>
constexpr ChainTable<D, P> make_chain_table() {
  ChainTable<D, P> t{};
  int h = 0;
  for (int k = 0; k <= P; ++k) {
    if (D == 2) {
      if (k == 0) {
        t.gi[h][0] = -1;
        t.ci[h] = 0;
        t.ph[h] = 0;
        t.deg[h] = 0;
        ++h;
      } else {
        for (int s = 0; s < 2; ++s) {
          t.gi[h][0] = -1;
          t.ci[h] = k;
          t.ph[h] = s == 0 ? 1 : -1;
          t.deg[h] = k;
          ++h;
        }
      }
      continue;
    }
    // Iterative enumeration of m_1 >= ... >= m_{D-2}, nested ascending loops.
    int m[D > 2 ? D - 1 : 1] = {};
    m[0] = k;
    int level = 1;
    for (int i = 1; i < D - 1; ++i) m[i] = 0;
    while (true) {
      // emit chain with m[1..D-2]
      const int last = m[D - 2];
      for (int s = 0; s < (last > 0 ? 2 : 1); ++s) {
        for (int l = 1; l <= D - 2; ++l) t.gi[h][l - 1] = g_index(P, l, m[l], m[l - 1] - m[l]);
        t.ci[h] = last;
        t.ph[h] = last == 0 ? 0 : (s == 0 ? 1 : -1);
        t.deg[h] = k;
        ++h;
      }
      // advance odometer from the deepest level
      level = D - 2;
      while (level >= 1) {
        if (m[level] < m[level - 1]) {
          ++m[level];
          for (int l = level + 1; l <= D - 2; ++l) m[l] = 0;
          break;
        }
        --level;
      }
      if (level < 1) break;
    }
  }
  return t;
}

// Raw (unnormalised) harmonic values Yraw[h] at relative position x (any
// scale, the direction is taken). For x = 0 every degree >= 1 vanishes and
// Yraw[0] = 1, which is the collocated-source rule of
// proj/src/expansion.cpp:273-289 once the norm is folded in.
// Number of chains in levels LEVEL..D-2 below m_{LEVEL-1} = mPrev.
constexpr int chain_count(int d, int level, int mPrev) {
  if (level == d - 2) return 2 * mPrev + 1;
  int c = 0;
  for (int m = 0; m <= mPrev; ++m) c += chain_count(d, level + 1, m);
  return c;
}

// Chain products for levels LEVEL..D-2 below a fixed prefix, generated by
// template recursion (nested ascending loops, the last level emitting +m then
// -m: the order of proj/src/harmonics.cpp:62-103). Every index is a template
// constant, so g/cA/cB/Y stay in registers.
template <int D, int P, int LEVEL, int MPREV, int M, int H0>
__device__ __forceinline__ void chain_products(double prod, const double* g, const double* cA, const double* cB,
                                               double* Y) {
  if constexpr (M <= MPREV) {
    const double pr = prod * g[g_index(P, LEVEL, M, MPREV - M)];
    if constexpr (LEVEL == D - 2) {
      Y[H0] = pr * cA[M];
      if constexpr (M > 0) Y[H0 + 1] = pr * cB[M];
      chain_products<D, P, LEVEL, MPREV, M + 1, H0 + (M > 0 ? 2 : 1)>(prod, g, cA, cB, Y);
    } else {
      chain_products<D, P, LEVEL + 1, M, 0, H0>(pr, g, cA, cB, Y);
      chain_products<D, P, LEVEL, MPREV, M + 1, H0 + chain_count(D, LEVEL + 1, M)>(prod, g, cA, cB, Y);
    }
  }
}

template <int D, int P, int K>
__device__ __forceinline__ void chain_degrees(const double* g, const double* cA, const double* cB, double* Y) {
  if constexpr (K <= P) {
    chain_products<D, P, 1, K, 0, harmonic_offset(D, K)>(1.0, g, cA, cB, Y);
    chain_degrees<D, P, K + 1>(g, cA, cB, Y);
  }
}

template <int D, int P>
__device__ __forceinline__ void harmonics_raw(const double (&x)[D], double r, double (&Y)[ChainTable<D, P>::H],
                                              double rinv = -1.0) {
  const double inv = rinv >= 0.0 ? rinv : (r > 0.0 ? 1.0 / r : 0.0);
  double v[D];
#pragma unroll
  for (int a = 0; a < D; ++a) v[a] = x[a] * inv;
  double cA[P + 1], cB[P + 1];
  cA[0] = 1.0;
  cB[0] = 0.0;
  const double cx = v[D - 2], cy = v[D - 1];
#pragma unroll
  for (int m = 1; m <= P; ++m) {
    cA[m] = cA[m - 1] * cx - cB[m - 1] * cy;
    cB[m] = cB[m - 1] * cx + cA[m - 1] * cy;
  }
  if constexpr (D == 2) {
    Y[0] = 1.0;
#pragma unroll
    for (int k = 1; k <= P; ++k) {
      Y[2 * k - 1] = cA[k];
      Y[2 * k] = cB[k];
    }
  } else {
    double tail[D - 1];
    {
      double acc = 0.0;
#pragma unroll
      for (int i = D - 1; i >= 0; --i) {
        acc += v[i] * v[i];
        if (i <= D - 2) tail[i] = acc;
      }
    }
    double g[(D - 2) * g_level_size(P)];
#pragma unroll
    for (int level = 1; level <= D - 2; ++level) {
      const double xx = v[level - 1];
      const double t2 = tail[level - 1];
#pragma unroll
      for (int m = 0; m <= P; ++m) {
        const int twoLam = D - 1 - level + 2 * m;  // 2 * lambda
        double* row = g + g_index(P, level, m, 0);
        row[0] = 1.0;
        if (P - m >= 1) row[1] = xx;
#pragma unroll
        for (int n = 2; n <= P - m; ++n)
          row[n] = fma(-gegen_beta(twoLam, n) * t2, row[n - 2], xx * row[n - 1]);
      }
    }
    chain_degrees<D, P, 0>(g, cA, cB, Y);
  }
}

}  // namespace fktb

#endif
