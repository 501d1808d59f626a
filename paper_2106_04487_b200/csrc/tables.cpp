// Plan-time host tables (see tables.hpp for the reference map).
#include "tables.hpp"

#include <cmath>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>

namespace fktb {

BigInt factorial(int n) {
  if (n < 0) throw std::invalid_argument("factorial: negative argument");
  BigInt f = 1;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

BigInt doubleFactorial(int n) {
  if (n < -1) throw std::invalid_argument("doubleFactorial: argument below -1");
  BigInt f = 1;
  for (int i = n; i >= 2; i -= 2) f *= i;
  return f;
}

BigInt binomial(int n, int k) {
  if (k < 0 || k > n || n < 0) return 0;
  k = std::min(k, n - k);
  BigInt b = 1;
  for (int i = 1; i <= k; ++i) {
    b *= n - k + i;
    b /= i;
  }
  return b;
}

BigInt intPow(BigInt base, int e) {
  BigInt p = 1;
  for (int i = 0; i < e; ++i) p *= base;
  return p;
}

Rational risingFactorial(const Rational& a, int n) {
  Rational p = 1, term = a;
  for (int i = 0; i < n; ++i) {
    p *= term;
    term += 1;
  }
  return p;
}

// ---------------------------------------------------------------------------
void Laurent::add(int power, const Rational& c) {
  if (c == Rational(0)) return;
  auto it = terms_.find(power);
  if (it == terms_.end()) {
    terms_.emplace(power, c);
  } else {
    it->second += c;
    if (it->second == Rational(0)) terms_.erase(it);
  }
}

Rational Laurent::coeff(int power) const {
  auto it = terms_.find(power);
  return it == terms_.end() ? Rational(0) : it->second;
}

Laurent Laurent::derivative() const {
  Laurent d;
  for (const auto& [p, c] : terms_)
    if (p != 0) d.add(p - 1, c * Rational(p));
  return d;
}

Laurent Laurent::operator+(const Laurent& o) const {
  Laurent r = *this;
  for (const auto& [p, c] : o.terms_) r.add(p, c);
  return r;
}

Laurent Laurent::operator*(const Laurent& o) const {
  Laurent r;
  for (const auto& [p1, c1] : terms_)
    for (const auto& [p2, c2] : o.terms_) r.add(p1 + p2, c1 * c2);
  return r;
}

// ---------------------------------------------------------------------------
namespace {

double param(const std::map<std::string, double>& p, const char* key, double fallback) {
  auto it = p.find(key);
  return it == p.end() ? fallback : it->second;
}

void checkParams(const std::string& name, const std::map<std::string, double>& given,
                 std::initializer_list<const char*> known) {
  for (const auto& kv : given) {
    bool ok = false;
    for (const char* k : known)
      if (kv.first == k) ok = true;
    if (!ok) throw std::invalid_argument("kernel '" + name + "': unknown parameter '" + kv.first + "'");
  }
}

}  // namespace

std::vector<std::string> builtinKernelNames() {
  return {"exponential", "matern12",  "matern32",   "cauchy",        "rational-quadratic",
          "gaussian",    "inverse-r", "inverse-r2", "inverse-r3",    "exp-over-r",
          "r-exp",       "cos-over-r", "exp-neg-inv-r", "exp-neg-inv-r2"};
}

// Reference proj/src/kernels.cpp:37-156: names, parameters, recurrences q
// (K' = qK) and value-at-zero conventions.
KernelSpec makeKernelSpec(const std::string& name, const std::map<std::string, double>& params) {
  KernelSpec k;
  k.name = name;
  k.params = params;
  const auto names = builtinKernelNames();
  for (std::size_t i = 0; i < names.size(); ++i)
    if (names[i] == name) k.id = static_cast<int>(i);
  if (k.id < 0) throw std::invalid_argument("unknown kernel '" + name + "'");
  switch (k.id) {
    case FKTB_KERNEL_EXPONENTIAL:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(-1), 0);
      k.valueAtZero = 1.0;
      break;
    case FKTB_KERNEL_MATERN12: {
      checkParams(name, params, {"sigma", "rho"});
      const double sigma = param(params, "sigma", 1.0);
      k.s2 = sigma * sigma;
      k.rho = param(params, "rho", 1.0);
      k.recurrence = Laurent::monomial(-Rational(1) / Rational(k.rho), 0);
      k.valueAtZero = k.s2;
      break;
    }
    case FKTB_KERNEL_MATERN32: {
      checkParams(name, params, {"sigma", "rho"});
      const double sigma = param(params, "sigma", 1.0);
      k.s2 = sigma * sigma;
      k.a = std::sqrt(3.0) / param(params, "rho", 1.0);
      k.valueAtZero = k.s2;
      break;
    }
    case FKTB_KERNEL_CAUCHY:
    case FKTB_KERNEL_RATIONAL_QUADRATIC: {
      checkParams(name, params, {"sigma"});
      const double sigma = param(params, "sigma", 1.0);
      k.is2 = 1.0 / (sigma * sigma);
      k.valueAtZero = 1.0;
      break;
    }
    case FKTB_KERNEL_GAUSSIAN:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(-2), 1);
      k.valueAtZero = 1.0;
      break;
    case FKTB_KERNEL_INVERSE_R:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(-1), -1);
      k.valueAtZero = 0.0;
      break;
    case FKTB_KERNEL_INVERSE_R2:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(-2), -1);
      k.valueAtZero = 0.0;
      break;
    case FKTB_KERNEL_INVERSE_R3:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(-3), -1);
      k.valueAtZero = 0.0;
      break;
    case FKTB_KERNEL_EXP_OVER_R: {
      checkParams(name, params, {});
      Laurent q;
      q.add(0, Rational(-1));
      q.add(-1, Rational(-1));
      k.recurrence = q;
      k.valueAtZero = 0.0;
      break;
    }
    case FKTB_KERNEL_R_EXP: {
      checkParams(name, params, {});
      Laurent q;
      q.add(-1, Rational(1));
      q.add(0, Rational(-1));
      k.recurrence = q;
      k.valueAtZero = 0.0;
      break;
    }
    case FKTB_KERNEL_COS_OVER_R:
      checkParams(name, params, {});
      k.valueAtZero = 0.0;
      break;
    case FKTB_KERNEL_EXP_NEG_INV_R:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(1), -2);
      k.valueAtZero = 0.0;
      break;
    case FKTB_KERNEL_EXP_NEG_INV_R2:
      checkParams(name, params, {});
      k.recurrence = Laurent::monomial(Rational(2), -3);
      k.valueAtZero = 0.0;
      break;
  }
  return k;
}

double kernelEvalHost(const KernelSpec& k, double r) {
  switch (k.id) {
    case FKTB_KERNEL_EXPONENTIAL: return std::exp(-r);
    case FKTB_KERNEL_MATERN12: return k.s2 * std::exp(-(r / k.rho));
    case FKTB_KERNEL_MATERN32: return k.s2 * (1.0 + k.a * r) * std::exp(-(k.a * r));
    case FKTB_KERNEL_CAUCHY: return 1.0 / (1.0 + r * r * k.is2);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return 1.0 / std::sqrt(1.0 + r * r * k.is2);
    case FKTB_KERNEL_GAUSSIAN: return std::exp(-(r * r));
    case FKTB_KERNEL_INVERSE_R: return 1.0 / r;
    case FKTB_KERNEL_INVERSE_R2: return 1.0 / (r * r);
    case FKTB_KERNEL_INVERSE_R3: return 1.0 / (r * r * r);
    case FKTB_KERNEL_EXP_OVER_R: return std::exp(-r) / r;
    case FKTB_KERNEL_R_EXP: return r * std::exp(-r);
    case FKTB_KERNEL_COS_OVER_R: return std::cos(r) / r;
    case FKTB_KERNEL_EXP_NEG_INV_R: return std::exp(-(1.0 / r));
    case FKTB_KERNEL_EXP_NEG_INV_R2: return std::exp(-(1.0 / (r * r)));
  }
  throw std::invalid_argument("kernelEvalHost: unknown kernel id");
}

// K on a jet argument (host; the formulas of kernelEvalHost in jet
// arithmetic, reference kernels.hpp:61-66).
fkt::Jet kernelJetHost(const KernelSpec& k, const fkt::Jet& r) {
  switch (k.id) {
    case FKTB_KERNEL_EXPONENTIAL: return exp(-r);
    case FKTB_KERNEL_MATERN12: return k.s2 * exp(-(r / k.rho));
    case FKTB_KERNEL_MATERN32: return k.s2 * ((1.0 + k.a * r) * exp(-(k.a * r)));
    case FKTB_KERNEL_CAUCHY: return reciprocal(1.0 + (r * r) * k.is2);
    case FKTB_KERNEL_RATIONAL_QUADRATIC: return pow(1.0 + (r * r) * k.is2, -0.5);
    case FKTB_KERNEL_GAUSSIAN: return exp(-(r * r));
    case FKTB_KERNEL_INVERSE_R: return reciprocal(r);
    case FKTB_KERNEL_INVERSE_R2: return reciprocal(r * r);
    case FKTB_KERNEL_INVERSE_R3: return reciprocal(r * r * r);
    case FKTB_KERNEL_EXP_OVER_R: return exp(-r) / r;
    case FKTB_KERNEL_R_EXP: return r * exp(-r);
    case FKTB_KERNEL_COS_OVER_R: return cos(r) / r;
    case FKTB_KERNEL_EXP_NEG_INV_R: return exp(-reciprocal(r));
    case FKTB_KERNEL_EXP_NEG_INV_R2: return exp(-reciprocal(r * r));
  }
  throw std::invalid_argument("kernelJetHost: unknown kernel id");
}

void fillKernelDesc(const KernelSpec& k, FktbKernelDesc& out) {
  out.id = k.id;
  out.pad_ = 0;
  out.s2 = k.s2;
  out.a = k.a;
  out.is2 = k.is2;
  out.rho = k.rho;
  out.diag = k.valueAtZero.value_or(0.0);
}

// ---------------------------------------------------------------------------
// Reference coefficients.cpp:12-17.
Rational bellCoefficient(int n, int m) {
  if (m < 1 || m > n) throw std::invalid_argument("bellCoefficient requires 1 <= m <= n");
  Rational r(doubleFactorial(2 * n - 2 * m - 1) * binomial(2 * n - m - 1, m - 1), intPow(2, n));
  if ((n + m) % 2 != 0) r = -r;
  return r;
}

// Reference coefficients.cpp:19-43 (d = 2 uses the Chebyshev limit).
std::vector<Rational> cosinePowerCoefficients(int d, int i) {
  if (d < 2 || i < 0) throw std::invalid_argument("cosinePowerCoefficients requires d >= 2, i >= 0");
  std::vector<Rational> out(static_cast<std::size_t>(i) + 1, Rational(0));
  for (int k = i % 2; k <= i; k += 2) {
    const int lo = (i - k) / 2, hi = (i + k) / 2;
    if (d == 2) {
      const BigInt num = k == 0 ? factorial(i) : factorial(i) * k;
      out[static_cast<std::size_t>(k)] = Rational(num, intPow(2, i) * factorial(lo) * factorial(hi));
    } else {
      const Rational alpha(d - 2, 2);
      const Rational num = Rational(factorial(i)) * (alpha + k);
      const Rational den = Rational(intPow(2, i) * factorial(lo)) * risingFactorial(alpha, hi + 1);
      out[static_cast<std::size_t>(k)] = num / den;
    }
  }
  return out;
}

// T-bar_kjm = sum_n binom(n, i) A_{k,i} (-2)^i / n! B_{n,m}, i = 2n - j
// (reference coefficients.cpp:52-95).
CoefTable::CoefTable(int d, int p) : d_(d), p_(p) {
  if (d < 2) throw std::invalid_argument("CoefficientTable requires d >= 2");
  if (p < 0) throw std::invalid_argument("CoefficientTable requires p >= 0");
  std::vector<std::vector<Rational>> bell(static_cast<std::size_t>(p) + 1), cosp(static_cast<std::size_t>(p) + 1);
  for (int n = 1; n <= p; ++n)
    for (int m = 1; m <= n; ++m) bell[static_cast<std::size_t>(n)].push_back(bellCoefficient(n, m));
  for (int i = 0; i <= p; ++i) cosp[static_cast<std::size_t>(i)] = cosinePowerCoefficients(d, i);
  layout();
  const std::size_t w = static_cast<std::size_t>(std::max(p, 1));
  for (int k = 0; k <= p; ++k)
    for (int j = k; j <= p; j += 2)
      for (int m = 1; m <= j; ++m) {
        Rational acc(0);
        for (int n = std::max((j + k + 1) / 2, m); n <= j; ++n) {
          const int i = 2 * n - j;
          if (i < k) continue;
          Rational term = Rational(binomial(n, i)) * cosp[static_cast<std::size_t>(i)][static_cast<std::size_t>(k)];
          term *= Rational(intPow(2, i), factorial(n));
          if (i % 2 != 0) term = -term;
          term *= bell[static_cast<std::size_t>(n)][static_cast<std::size_t>(m - 1)];
          acc += term;
        }
        t_[row(k, j) * w + static_cast<std::size_t>(m - 1)] = acc;
      }
  td_.resize(t_.size());
  for (std::size_t i = 0; i < t_.size(); ++i) td_[i] = toDouble(t_[i]);
}

void CoefTable::layout() {
  rowOffset_.assign(static_cast<std::size_t>(p_) + 2, 0);
  std::size_t rows = 0;
  for (int k = 0; k <= p_; ++k) {
    rowOffset_[static_cast<std::size_t>(k)] = rows;
    rows += static_cast<std::size_t>((p_ - k) / 2) + 1;
  }
  rowOffset_[static_cast<std::size_t>(p_) + 1] = rows;
  t_.assign(rows * static_cast<std::size_t>(std::max(p_, 1)), Rational(0));
}

std::string CoefTable::serialize() const {
  std::ostringstream os;
  os << "fkt-tbar 1 " << d_ << " " << p_ << "\n";
  for (int k = 0; k <= p_; ++k)
    for (int j = k; j <= p_; j += 2)
      for (int m = 1; m <= j; ++m) {
        const Rational& q = tbar(k, j, m);
        os << k << " " << j << " " << m << " " << q.num() << " " << q.den() << "\n";
      }
  return os.str();
}

std::optional<CoefTable> CoefTable::deserialize(const std::string& text) {
  std::istringstream is(text);
  std::string magic;
  int version = 0, d = 0, p = 0;
  if (!(is >> magic >> version >> d >> p) || magic != "fkt-tbar" || version != 1) return std::nullopt;
  if (d < 2 || p < 0 || p > kMaxInternalOrder) return std::nullopt;
  CoefTable t;
  t.d_ = d;
  t.p_ = p;
  t.layout();
  const std::size_t w = static_cast<std::size_t>(std::max(p, 1));
  int k, j, m;
  BigInt num, den;
  std::size_t count = 0;
  while (is >> k >> j >> m >> num >> den) {
    if (den.isZero()) return std::nullopt;
    if (k < 0 || j < k || j > p || m < 1 || m > j || (j - k) % 2 != 0) return std::nullopt;
    t.t_[t.row(k, j) * w + static_cast<std::size_t>(m - 1)] = Rational(num, den);
    ++count;
  }
  std::size_t expected = 0;
  for (int kk = 0; kk <= p; ++kk)
    for (int jj = kk; jj <= p; jj += 2) expected += static_cast<std::size_t>(jj);
  if (count != expected) return std::nullopt;
  t.td_.resize(t.t_.size());
  for (std::size_t i = 0; i < t.t_.size(); ++i) t.td_[i] = toDouble(t.t_[i]);
  return t;
}

const Rational& CoefTable::tbar(int k, int j, int m) const {
  static const Rational kZero(0);
  if (k < 0 || j < k || j > p_ || m < 1 || m > j || (j - k) % 2 != 0) return kZero;
  return t_[row(k, j) * static_cast<std::size_t>(std::max(p_, 1)) + static_cast<std::size_t>(m - 1)];
}

double CoefTable::tbarDouble(int k, int j, int m) const {
  if (k < 0 || j < k || j > p_ || m < 1 || m > j || (j - k) % 2 != 0) return 0.0;
  return td_[row(k, j) * static_cast<std::size_t>(std::max(p_, 1)) + static_cast<std::size_t>(m - 1)];
}

const CoefTable& coefTable(int d, int p) {
  if (p > kMaxExpansionOrder) throw std::invalid_argument("expansion order " + std::to_string(p) +
                                                          " exceeds the supported cap " +
                                                          std::to_string(kMaxExpansionOrder));
  static std::mutex mutex;
  static std::map<std::pair<int, int>, std::unique_ptr<CoefTable>> tables;
  std::lock_guard<std::mutex> lock(mutex);
  auto& e = tables[{d, p}];
  if (!e) {
    // reference coefficients.cpp:170-214 (FKT_CACHE_DIR)
    const char* dir = std::getenv("FKT_CACHE_DIR");
    std::optional<std::filesystem::path> file;
    if (dir && *dir)
      file = std::filesystem::path(dir) / ("fkt-tbar-v1-d" + std::to_string(d) + "-p" + std::to_string(p) + ".txt");
    if (file) {
      std::ifstream in(*file);
      if (in) {
        std::stringstream buf;
        buf << in.rdbuf();
        if (auto loaded = CoefTable::deserialize(buf.str())) e = std::make_unique<CoefTable>(std::move(*loaded));
      }
    }
    if (!e) {
      e = std::make_unique<CoefTable>(d, p);
      if (file) {
        std::error_code ec;
        std::filesystem::create_directories(file->parent_path(), ec);
        std::ofstream out(*file);
        if (out) out << e->serialize();
      }
    }
  }
  return *e;
}

std::size_t expansionSize(int d, int p) {
  if (d < 2 || p < 0) throw std::invalid_argument("expansionSize requires d >= 2, p >= 0");
  return binomial(d + p, p).convert_to<std::size_t>();
}

// ---------------------------------------------------------------------------
namespace {

constexpr double kPi = 3.14159265358979323846;

double sphereSurface(int d) { return 2.0 * std::pow(kPi, 0.5 * d) / std::tgamma(0.5 * d); }

double gegenbauerNormSq(int n, double lambda) {
  const double logNum = std::log(kPi) + (1.0 - 2.0 * lambda) * std::log(2.0) + std::lgamma(n + 2.0 * lambda);
  const double logDen = std::lgamma(n + 1.0) + std::log(n + lambda) + 2.0 * std::lgamma(lambda);
  return std::exp(logNum - logDen);
}

// Chain enumeration order of reference harmonics.cpp:62-103: nested levels
// m_1 >= m_2 >= ... ascending, the last level emitting +m then -m.
void enumerate(int levelsLeft, int top, std::vector<int>& prefix, std::vector<std::vector<int>>& out) {
  if (levelsLeft == 1) {
    for (int m = 0; m <= top; ++m) {
      prefix.push_back(m);
      out.push_back(prefix);
      prefix.pop_back();
      if (m > 0) {
        prefix.push_back(-m);
        out.push_back(prefix);
        prefix.pop_back();
      }
    }
    return;
  }
  for (int m = 0; m <= top; ++m) {
    prefix.push_back(m);
    enumerate(levelsLeft - 1, m, prefix, out);
    prefix.pop_back();
  }
}

}  // namespace

double gegenbauerAtOne(int d, int k) {
  if (d == 2) return k == 0 ? 1.0 : 2.0 / k;
  return toDouble(Rational(binomial(k + d - 3, k)));
}

std::size_t harmonicIndexCount(int d, int k) {
  if (d < 2 || k < 0) throw std::invalid_argument("harmonicIndexCount requires d >= 2, k >= 0");
  BigInt c = binomial(k + d - 1, k) - binomial(k + d - 3, k - 2);
  return c.convert_to<std::size_t>();
}

double additionNormalizer(int d, int k) {
  return sphereSurface(d) * gegenbauerAtOne(d, k) / static_cast<double>(harmonicIndexCount(d, k));
}

// Reference harmonics.cpp:118-158.
HarmonicStructure::HarmonicStructure(int d, int p) : d_(d), p_(p) {
  if (d < 2) throw std::invalid_argument("HarmonicBasis requires d >= 2");
  if (p < 0) throw std::invalid_argument("HarmonicBasis requires maxDegree >= 0");
  offset_.assign(static_cast<std::size_t>(p) + 2, 0);
  z_.resize(static_cast<std::size_t>(p) + 1);
  chains_.resize(static_cast<std::size_t>(p) + 1);
  std::size_t off = 0;
  for (int k = 0; k <= p; ++k) {
    offset_[static_cast<std::size_t>(k)] = off;
    z_[static_cast<std::size_t>(k)] = additionNormalizer(d, k);
    std::vector<std::vector<int>> raw;
    if (d == 2) {
      if (k == 0)
        raw.push_back({0});
      else {
        raw.push_back({k});
        raw.push_back({-k});
      }
    } else {
      std::vector<int> prefix;
      enumerate(d - 2, k, prefix, raw);
    }
    for (const auto& rc : raw) {
      HarmonicChain c;
      c.m.resize(rc.size() + 1);
      c.m[0] = k;
      for (std::size_t i = 0; i < rc.size(); ++i) c.m[i + 1] = std::abs(rc[i]);
      c.phase = rc.back() > 0 ? 1 : (rc.back() < 0 ? -1 : 0);
      if (d == 2) {
        c.norm = 1.0 / std::sqrt(c.phase == 0 ? 2.0 * kPi : kPi);
        c.m.resize(1);
      } else {
        double norm = 1.0;
        for (int level = 1; level <= d - 2; ++level) {
          const double lambda = 0.5 * (d - 1 - level) + c.m[static_cast<std::size_t>(level)];
          const int n = c.m[static_cast<std::size_t>(level - 1)] - c.m[static_cast<std::size_t>(level)];
          norm /= gegenbauerNormSq(n, lambda);
        }
        norm /= (c.phase == 0 ? 2.0 * kPi : kPi);
        c.norm = std::sqrt(norm);
      }
      chains_[static_cast<std::size_t>(k)].push_back(std::move(c));
    }
    off += chains_[static_cast<std::size_t>(k)].size();
  }
  offset_[static_cast<std::size_t>(p) + 1] = off;
  total_ = off;
}

// ---------------------------------------------------------------------------
namespace {

struct RatMat {
  int rows, cols;
  std::vector<Rational> a;
  RatMat(int r, int c) : rows(r), cols(c), a(static_cast<std::size_t>(r) * c) {}
  Rational& at(int i, int j) { return a[static_cast<std::size_t>(i) * cols + j]; }
};

// Gram-Schmidt with exact largest-norm column pivoting, unnormalised
// (reference expansion.cpp:116-173). Returns rank; q columns and r rows.
int rankRevealingQr(RatMat& m, std::vector<std::vector<Rational>>& qCols, std::vector<std::vector<Rational>>& rRows) {
  const int rows = m.rows, cols = m.cols;
  std::vector<std::vector<Rational>> work(static_cast<std::size_t>(cols), std::vector<Rational>(static_cast<std::size_t>(rows)));
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) work[static_cast<std::size_t>(j)][static_cast<std::size_t>(i)] = m.at(i, j);
  std::vector<bool> used(static_cast<std::size_t>(cols), false);
  for (int step = 0; step < std::min(rows, cols); ++step) {
    int pivot = -1;
    Rational best(0);
    for (int j = 0; j < cols; ++j) {
      if (used[static_cast<std::size_t>(j)]) continue;
      Rational norm(0);
      for (const Rational& x : work[static_cast<std::size_t>(j)]) norm += x * x;
      if (pivot < 0 || norm > best) {
        best = norm;
        pivot = j;
      }
    }
    if (pivot < 0 || best == Rational(0)) break;
    used[static_cast<std::size_t>(pivot)] = true;
    std::vector<Rational> q = work[static_cast<std::size_t>(pivot)];
    std::vector<Rational> rRow(static_cast<std::size_t>(cols), Rational(0));
    rRow[static_cast<std::size_t>(pivot)] = 1;
    for (int j = 0; j < cols; ++j) {
      if (used[static_cast<std::size_t>(j)]) continue;
      Rational proj(0);
      for (int i = 0; i < rows; ++i) proj += q[static_cast<std::size_t>(i)] * work[static_cast<std::size_t>(j)][static_cast<std::size_t>(i)];
      proj /= best;
      if (proj == Rational(0)) continue;
      rRow[static_cast<std::size_t>(j)] = proj;
      for (int i = 0; i < rows; ++i) work[static_cast<std::size_t>(j)][static_cast<std::size_t>(i)] -= proj * q[static_cast<std::size_t>(i)];
    }
    qCols.push_back(std::move(q));
    rRows.push_back(std::move(rRow));
  }
  return static_cast<int>(qCols.size());
}

}  // namespace

// Reference expansion.cpp:179-243: coefficient matrix of K(r) r^s r'^j in the
// degree-k radial function, exact QR, factors F_i (Laurent in r) and G_i
// (polynomial in r').
std::vector<RadialFactor> radialCompression(const KernelSpec& kernel, const CoefTable& table, int p) {
  if (!kernel.recurrence) throw NotRecurrenceKernelError(kernel.name);
  const Laurent& q = *kernel.recurrence;
  std::vector<Laurent> lau(static_cast<std::size_t>(p) + 1);
  lau[0] = Laurent::monomial(Rational(1), 0);
  for (int m = 1; m <= p; ++m) lau[static_cast<std::size_t>(m)] = lau[static_cast<std::size_t>(m - 1)].derivative() + lau[static_cast<std::size_t>(m - 1)] * q;

  std::vector<RadialFactor> out;
  for (int k = 0; k <= p; ++k) {
    std::map<int, std::map<int, Rational>> coeffs;
    for (int j = k; j <= p; j += 2) {
      for (int m = 1; m <= j; ++m) {
        const Rational& t = table.tbar(k, j, m);
        if (t == Rational(0)) continue;
        for (const auto& [power, c] : lau[static_cast<std::size_t>(m)].terms()) coeffs[power + m - j][j] += c * t;
      }
      if (k == 0 && j == 0) coeffs[0][0] += 1;
    }
    std::vector<int> rPowers, srcPowers;
    for (const auto& kv : coeffs) rPowers.push_back(kv.first);
    for (int j = k; j <= p; j += 2) srcPowers.push_back(j);
    RatMat mat(static_cast<int>(rPowers.size()), static_cast<int>(srcPowers.size()));
    for (std::size_t i = 0; i < rPowers.size(); ++i) {
      const auto& row = coeffs[rPowers[i]];
      for (std::size_t j = 0; j < srcPowers.size(); ++j) {
        auto it = row.find(srcPowers[j]);
        mat.at(static_cast<int>(i), static_cast<int>(j)) = it == row.end() ? Rational(0) : it->second;
      }
    }
    std::vector<std::vector<Rational>> qCols, rRows;
    const int rank = rankRevealingQr(mat, qCols, rRows);
    RadialFactor f;
    f.degree = k;
    f.rank = rank;
    for (int t = 0; t < rank; ++t) {
      Laurent fr, gs;
      for (std::size_t i = 0; i < rPowers.size(); ++i) fr.add(rPowers[i], qCols[static_cast<std::size_t>(t)][i]);
      for (std::size_t j = 0; j < srcPowers.size(); ++j) gs.add(srcPowers[j], rRows[static_cast<std::size_t>(t)][j]);
      f.target.push_back(std::move(fr));
      f.source.push_back(std::move(gs));
    }
    out.push_back(std::move(f));
  }
  return out;
}

}  // namespace fktb
