// Host tables for the monomial-moment S2M (see moments.hpp).
#include "moments.hpp"

#include <algorithm>

#include "cart_layout.hpp"

#include <map>
#include <stdexcept>

namespace fktb {
namespace {

void enumerate(int d, int dim, int rem, std::vector<int>& cur, std::vector<std::vector<int>>& out) {
  if (dim == d) {
    out.push_back(cur);
    return;
  }
  for (int e = 0; e <= rem; ++e) {
    cur[static_cast<std::size_t>(dim)] = e;
    enumerate(d, dim + 1, rem - e, cur, out);
  }
  cur[static_cast<std::size_t>(dim)] = 0;
}

struct PolyAlgebra {
  const MonomialBasis& B;
  std::map<std::vector<int>, int> idx;
  explicit PolyAlgebra(const MonomialBasis& b) : B(b) {
    for (int i = 0; i < B.count(); ++i) idx[B.exps[static_cast<std::size_t>(i)]] = i;
  }
  using Poly = std::vector<double>;
  Poly zero() const { return Poly(static_cast<std::size_t>(B.count()), 0.0); }
  Poly one() const {
    Poly r = zero();
    r[0] = 1.0;  // the all-zero exponent is enumerated first
    return r;
  }
  Poly var(int i) const {
    Poly r = zero();
    std::vector<int> a(static_cast<std::size_t>(B.d), 0);
    a[static_cast<std::size_t>(i)] = 1;
    r[static_cast<std::size_t>(idx.at(a))] = 1.0;
    return r;
  }
  Poly mul(const Poly& x, const Poly& y) const {
    Poly r = zero();
    std::vector<int> a(static_cast<std::size_t>(B.d));
    for (int i = 0; i < B.count(); ++i) {
      if (x[static_cast<std::size_t>(i)] == 0.0) continue;
      for (int j = 0; j < B.count(); ++j) {
        if (y[static_cast<std::size_t>(j)] == 0.0) continue;
        int deg = 0;
        for (int q = 0; q < B.d; ++q) {
          a[static_cast<std::size_t>(q)] = B.exps[static_cast<std::size_t>(i)][static_cast<std::size_t>(q)] +
                                           B.exps[static_cast<std::size_t>(j)][static_cast<std::size_t>(q)];
          deg += a[static_cast<std::size_t>(q)];
        }
        if (deg > B.p) throw std::logic_error("monomial moments: degree overflow");
        r[static_cast<std::size_t>(idx.at(a))] += x[static_cast<std::size_t>(i)] * y[static_cast<std::size_t>(j)];
      }
    }
    return r;
  }
  static Poly axpby(double a, const Poly& x, double b, const Poly& y) {
    Poly r(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) r[i] = a * x[i] + b * y[i];
    return r;
  }
};

double binom(int n, int k) {
  double b = 1.0;
  for (int i = 1; i <= k; ++i) b = b * (n - k + i) / i;
  return b;
}

}  // namespace

MonomialBasis::MonomialBasis(int d_, int p_) : d(d_), p(p_) {
  std::vector<int> cur(static_cast<std::size_t>(d), 0);
  enumerate(d, 0, p, cur, exps);
}

int MonomialBasis::index(const std::vector<int>& a) const {
  for (int i = 0; i < count(); ++i)
    if (exps[static_cast<std::size_t>(i)] == a) return i;
  return -1;
}

MomentTables buildMomentTables(int d, int p, const HarmonicStructure& hs, const std::vector<RadialFactor>& factors,
                               bool compressed, const std::vector<double>& hscale) {
  const MonomialBasis B(d, p);
  const PolyAlgebra alg(B);
  using Poly = PolyAlgebra::Poly;
  MomentTables out;
  out.count = B.count();

  // Solid harmonics S_h (the device's raw chain products times |x|^k),
  // built with the same recurrences (harmonics.cpp:172-230) symbolically.
  std::vector<Poly> cA(static_cast<std::size_t>(p) + 1), cB(static_cast<std::size_t>(p) + 1);
  cA[0] = alg.one();
  cB[0] = alg.zero();
  const Poly cx = alg.var(d - 2), cy = alg.var(d - 1);
  for (int m = 1; m <= p; ++m) {
    cA[static_cast<std::size_t>(m)] = PolyAlgebra::axpby(1.0, alg.mul(cA[static_cast<std::size_t>(m - 1)], cx), -1.0,
                                                          alg.mul(cB[static_cast<std::size_t>(m - 1)], cy));
    cB[static_cast<std::size_t>(m)] = PolyAlgebra::axpby(1.0, alg.mul(cB[static_cast<std::size_t>(m - 1)], cx), 1.0,
                                                          alg.mul(cA[static_cast<std::size_t>(m - 1)], cy));
  }
  // g[level][m][n]
  std::vector<std::vector<std::vector<Poly>>> g(static_cast<std::size_t>(std::max(d - 1, 1)));
  for (int level = 1; level <= d - 2; ++level) {
    Poly tail = alg.zero();
    for (int i = level - 1; i < d; ++i) {
      const Poly xi = alg.var(i);
      tail = PolyAlgebra::axpby(1.0, tail, 1.0, alg.mul(xi, xi));
    }
    const Poly xx = alg.var(level - 1);
    auto& byM = g[static_cast<std::size_t>(level)];
    byM.resize(static_cast<std::size_t>(p) + 1);
    for (int m = 0; m <= p; ++m) {
      const int twoLam = d - 1 - level + 2 * m;
      auto& row = byM[static_cast<std::size_t>(m)];
      row.resize(static_cast<std::size_t>(p - m) + 1);
      row[0] = alg.one();
      if (p - m >= 1) row[1] = PolyAlgebra::axpby(static_cast<double>(twoLam), xx, 0.0, xx);
      for (int nn = 2; nn <= p - m; ++nn)
        row[static_cast<std::size_t>(nn)] =
            PolyAlgebra::axpby(static_cast<double>(2 * nn + twoLam - 2) / nn, alg.mul(xx, row[static_cast<std::size_t>(nn - 1)]),
                               -static_cast<double>(nn + twoLam - 2) / nn, alg.mul(tail, row[static_cast<std::size_t>(nn - 2)]));
    }
  }
  std::vector<Poly> S(hs.total());
  for (int k = 0; k <= p; ++k) {
    std::size_t h = hs.degreeOffset(k);
    for (const HarmonicChain& ch : hs.chains(k)) {
      if (d == 2) {
        S[h] = k == 0 ? alg.one() : (ch.phase >= 0 ? cA[static_cast<std::size_t>(k)] : cB[static_cast<std::size_t>(k)]);
      } else {
        Poly prod = ch.phase >= 0 ? cA[static_cast<std::size_t>(ch.m[static_cast<std::size_t>(d - 2)])]
                                  : cB[static_cast<std::size_t>(ch.m[static_cast<std::size_t>(d - 2)])];
        for (int level = 1; level <= d - 2; ++level) {
          const int mi = ch.m[static_cast<std::size_t>(level)], nn = ch.m[static_cast<std::size_t>(level - 1)] - mi;
          prod = alg.mul(prod, g[static_cast<std::size_t>(level)][static_cast<std::size_t>(mi)][static_cast<std::size_t>(nn)]);
        }
        S[h] = prod;
      }
      ++h;
    }
  }
  // |x|^(2s) powers
  Poly r2 = alg.zero();
  for (int i = 0; i < d; ++i) r2 = PolyAlgebra::axpby(1.0, r2, 1.0, alg.mul(alg.var(i), alg.var(i)));
  std::vector<Poly> r2s(static_cast<std::size_t>(p / 2) + 1);
  r2s[0] = alg.one();
  for (std::size_t s = 1; s < r2s.size(); ++s) r2s[s] = alg.mul(r2s[s - 1], r2);

  // T rows in the padded (k, s, h) layout.
  int P = 0;
  std::vector<int> cOff(static_cast<std::size_t>(p) + 2);
  for (int k = 0; k <= p; ++k) {
    cOff[static_cast<std::size_t>(k)] = P;
    P += static_cast<int>(hs.degreeCount(k)) * ((p - k) / 2 + 1);
  }
  out.T.assign(static_cast<std::size_t>(P) * out.count, 0.0);
  for (int k = 0; k <= p; ++k) {
    const int nh = static_cast<int>(hs.degreeCount(k));
    const int su = (p - k) / 2 + 1;
    for (int hh = 0; hh < nh; ++hh) {
      const std::size_t h = hs.degreeOffset(k) + static_cast<std::size_t>(hh);
      for (int s = 0; s < su; ++s) {
        Poly row = alg.zero();
        if (!compressed) {
          row = alg.mul(r2s[static_cast<std::size_t>(s)], S[h]);
        } else {
          const RadialFactor& f = factors[static_cast<std::size_t>(k)];
          if (s >= f.rank) continue;
          for (const auto& [pw, c] : f.source[static_cast<std::size_t>(s)].terms()) {
            const int sj = (pw - k) / 2;  // source power r'^pw = |x|^(pw-k) * |x|^k
            row = PolyAlgebra::axpby(1.0, row, toDouble(c), alg.mul(r2s[static_cast<std::size_t>(sj)], S[h]));
          }
        }
        const std::size_t c = static_cast<std::size_t>(cOff[static_cast<std::size_t>(k)] + s * nh + hh);
        for (int a = 0; a < out.count; ++a) out.T[c * out.count + static_cast<std::size_t>(a)] = hscale[h] * row[static_cast<std::size_t>(a)];
      }
    }
  }

  // Shift table (multinomial binomial theorem), CSR over the output monomial.
  out.off.assign(static_cast<std::size_t>(out.count) + 1, 0);
  for (int a = 0; a < out.count; ++a) {
    out.off[static_cast<std::size_t>(a)] = static_cast<int>(out.b.size());
    const auto& ea = B.exps[static_cast<std::size_t>(a)];
    for (int bb = 0; bb < out.count; ++bb) {
      const auto& eb = B.exps[static_cast<std::size_t>(bb)];
      bool le = true;
      double coef = 1.0;
      std::vector<int> gam(static_cast<std::size_t>(d));
      for (int q = 0; q < d && le; ++q) {
        if (eb[static_cast<std::size_t>(q)] > ea[static_cast<std::size_t>(q)]) le = false;
        gam[static_cast<std::size_t>(q)] = ea[static_cast<std::size_t>(q)] - eb[static_cast<std::size_t>(q)];
        if (le) coef *= binom(ea[static_cast<std::size_t>(q)], eb[static_cast<std::size_t>(q)]);
      }
      if (!le) continue;
      out.b.push_back(bb);
      out.g.push_back(alg.idx.at(gam));
      out.coef.push_back(coef);
    }
  }
  out.off[static_cast<std::size_t>(out.count)] = static_cast<int>(out.b.size());
  return out;
}

// ---------------------------------------------------------------------------
// Cartesian M2T table (see moments.hpp, cart_layout.hpp).
namespace {

// Exponent tuples of the monomials with total degree in [lo, hi] over
// variables 0..nv-1, in the order of the device recursion (far.cu cart_eval):
// the last variable's power descending, recursively; x_0's power descending.
void cartEnumerate(int nv, int lo, int hi, std::vector<int>& cur, std::vector<std::vector<int>>& out) {
  if (nv == 1) {
    for (int j = hi; j >= lo; --j) {
      cur[0] = j;
      out.push_back(cur);
    }
    cur[0] = 0;
    return;
  }
  for (int e = hi; e >= 0; --e) {
    cur[static_cast<std::size_t>(nv) - 1] = e;
    cartEnumerate(nv - 1, std::max(lo - e, 0), hi - e, cur, out);
  }
  cur[static_cast<std::size_t>(nv) - 1] = 0;
}

double factorialD(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

double multinomialD(const std::vector<int>& a) {
  int n = 0;
  for (int v : a) n += v;
  double r = factorialD(n);
  for (int v : a) r /= factorialD(v);
  return r;
}

}  // namespace

bool cartSupported(int kid, int d, int p) {
  if (kid != FKTB_KERNEL_MATERN32 && kid != FKTB_KERNEL_GAUSSIAN && kid != FKTB_KERNEL_CAUCHY &&
      kid != FKTB_KERNEL_MATERN12 && kid != FKTB_KERNEL_EXPONENTIAL)
    return false;
  switch (d * 100 + p) {  // the compiled shapes (far.cu launchCart)
    case 304:
    case 306:
    case 308:
    case 504: return true;
    default: return false;
  }
}

std::vector<double> buildCartTable(int d, int p, const FktbKernelDesc& kernel, int& PCart) {
  PCart = 0;
  if (!cartSupported(kernel.id, d, p)) return {};
  const MonomialBasis B(d, p);
  std::map<std::vector<int>, int> idx;
  for (int i = 0; i < B.count(); ++i) idx[B.exps[static_cast<std::size_t>(i)]] = i;
  const int C = B.count();
  // constant factor of F^(n)(q)/n! (the q-dependent factor is evaluated per pair)
  auto factor = [&](int n) {
    if (kernel.id == FKTB_KERNEL_GAUSSIAN) return ((n & 1) ? -1.0 : 1.0) / factorialD(n);  // F = e^-q
    if (kernel.id == FKTB_KERNEL_CAUCHY) {  // F = 1 / (1 + is2 q): F^(n)/n! = (-is2)^n F^(n+1)
      double f = 1.0;
      for (int i = 0; i < n; ++i) f *= -kernel.is2;
      return f;
    }
    // Matern-3/2 and e^(-a r) (Matern-1/2, exponential): F^(n) = s2 (a^2/2)^n (-1)^n h_n(u),
    // u = a sqrt(q) (far.cu m2t_cart)
    const double a = kernel.id == FKTB_KERNEL_MATERN32 ? kernel.a : kernel.id == FKTB_KERNEL_MATERN12 ? 1.0 / kernel.rho : 1.0;
    double f = (kernel.id == FKTB_KERNEL_EXPONENTIAL ? 1.0 : kernel.s2) / factorialD(n);
    for (int i = 0; i < n; ++i) f *= -0.5 * a * a;
    return f;
  };
  const bool merged = cart_merged(kernel.id);
  PCart = cart_total(kernel.id, d, p);
  std::vector<double> T(static_cast<std::size_t>(PCart) * C, 0.0);
  std::map<std::vector<int>, int> mergedRow;
  if (merged) {
    std::vector<std::vector<int>> order;
    std::vector<int> cur(static_cast<std::size_t>(d), 0);
    cartEnumerate(d, 0, p, cur, order);
    for (std::size_t r = 0; r < order.size(); ++r) mergedRow[order[r]] = static_cast<int>(r);
  }
  for (int n = 0; n <= p; ++n) {
    std::vector<std::vector<int>> order;
    std::vector<int> cur(static_cast<std::size_t>(d), 0);
    cartEnumerate(d, cart_block_lo(p, n), n, cur, order);
    const int base = merged ? 0 : cart_block_offset(kernel.id, d, p, n);
    for (std::size_t r = 0; r < order.size(); ++r) {
      const std::vector<int>& beta = order[r];
      int a = 0;
      for (int v : beta) a += v;
      const int i = n - a;  // this term carries |x'|^(2i)
      // F-factor * binom(n, i) (-2)^a (a!/beta!) * nu_{i,beta},
      // nu_{i,beta} = sum_{|gamma| = i} (i!/gamma!) mu_{beta + 2 gamma}
      double c = factor(n) * multinomialD(beta);
      for (int k = 1; k <= i; ++k) c = c * (n - i + k) / k;
      for (int k = 0; k < a; ++k) c *= -2.0;
      const int row = merged ? mergedRow.at(beta) : base + static_cast<int>(r);
      for (int g = 0; g < C; ++g) {
        const std::vector<int>& gamma = B.exps[static_cast<std::size_t>(g)];
        int gs = 0;
        for (int v : gamma) gs += v;
        if (gs != i) continue;
        std::vector<int> al(static_cast<std::size_t>(d));
        for (int q = 0; q < d; ++q)
          al[static_cast<std::size_t>(q)] = beta[static_cast<std::size_t>(q)] + 2 * gamma[static_cast<std::size_t>(q)];
        T[static_cast<std::size_t>(row) * C + static_cast<std::size_t>(idx.at(al))] += c * multinomialD(gamma);
      }
    }
  }
  return T;
}

}  // namespace fktb
