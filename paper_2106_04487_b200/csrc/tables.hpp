// Plan-time host tables for the FKT expansion (product code, host C++).
//
// Restates, in this repo's own code, the kernel registry
// (reference proj/src/kernels.cpp:37-163), the exact coefficient table T-bar
// (proj/src/coefficients.cpp:12-111), the hyperspherical-harmonic chain
// structure and normalisers (proj/src/harmonics.cpp:35-158) and the exact
// radial compression (proj/src/expansion.cpp:116-243). Everything here runs
// once per plan on the host and is uploaded to the device (kernel parameter
// space) by plan.cpp.
#ifndef FKTB_TABLES_HPP
#define FKTB_TABLES_HPP

#include "fkt/jet.hpp"
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "exact.hpp"
#include "fkt_device_types.h"

namespace fktb {

using exact::BigInt;
using exact::Rational;

inline double toDouble(const Rational& q) { return q.convert_to<double>(); }
BigInt factorial(int n);
BigInt doubleFactorial(int n);
BigInt binomial(int n, int k);
BigInt intPow(BigInt base, int e);
Rational risingFactorial(const Rational& a, int n);

// Sparse Laurent polynomial with exact coefficients (reference
// proj/include/fkt/laurent.hpp:17-95).
class Laurent {
 public:
  static Laurent monomial(const Rational& c, int power) {
    Laurent l;
    l.add(power, c);
    return l;
  }
  void add(int power, const Rational& c);
  Rational coeff(int power) const;
  const std::map<int, Rational>& terms() const { return terms_; }
  bool empty() const { return terms_.empty(); }
  int minPower() const { return terms_.empty() ? 0 : terms_.begin()->first; }
  int maxPower() const { return terms_.empty() ? 0 : terms_.rbegin()->first; }
  Laurent derivative() const;
  Laurent operator+(const Laurent& o) const;
  Laurent operator*(const Laurent& o) const;
  bool operator==(const Laurent& o) const { return terms_ == o.terms_; }

 private:
  std::map<int, Rational> terms_;
};

// ---------------------------------------------------------------------------
// Kernel registry: the 14 built-in isotropic kernels by name.
struct KernelSpec {
  int id = -1;  // FKTB_KERNEL_* (fkt_device_types.h)
  std::string name;
  std::map<std::string, double> params;
  double s2 = 1.0, a = 1.0, is2 = 1.0, rho = 1.0;
  std::optional<Laurent> recurrence;  // K' = q K (exact rational q)
  std::optional<double> valueAtZero;
};

KernelSpec makeKernelSpec(const std::string& name, const std::map<std::string, double>& params);
std::vector<std::string> builtinKernelNames();
// K(r) for r > 0 (host), same formula as the device evaluator.
double kernelEvalHost(const KernelSpec& k, double r);
// K on a jet argument (host).
fkt::Jet kernelJetHost(const KernelSpec& k, const fkt::Jet& r);
void fillKernelDesc(const KernelSpec& k, FktbKernelDesc& out);

// ---------------------------------------------------------------------------
constexpr int kMaxExpansionOrder = 20;  // reference coefficients.hpp:31

Rational bellCoefficient(int n, int m);
std::vector<Rational> cosinePowerCoefficients(int d, int i);

class CoefTable {
 public:
  CoefTable(int d, int p);
  int dimension() const { return d_; }
  int maxOrder() const { return p_; }
  const Rational& tbar(int k, int j, int m) const;
  double tbarDouble(int k, int j, int m) const;

  // Text format of the reference (coefficients.cpp:113-166): header
  // "fkt-tbar 1 d p", then one "k j m num den" line per entry. deserialize
  // returns nullopt on anything malformed, as the reference does.
  std::string serialize() const;
  static std::optional<CoefTable> deserialize(const std::string& text);
  bool operator==(const CoefTable& o) const { return d_ == o.d_ && p_ == o.p_ && t_ == o.t_; }

 private:
  CoefTable() = default;
  void layout();
  std::size_t row(int k, int j) const { return rowOffset_[static_cast<std::size_t>(k)] + static_cast<std::size_t>((j - k) / 2); }
  int d_ = 0, p_ = 0;
  std::vector<Rational> t_;
  std::vector<double> td_;
  std::vector<std::size_t> rowOffset_;
};

// Memoised, mutex-guarded (reference coefficients.cpp:187-220); honours the
// reference's FKT_CACHE_DIR on-disk cache (file fkt-tbar-v1-d<d>-p<p>.txt in
// the serialize() format, read if it parses, written after a build).
const CoefTable& coefTable(int d, int p);
constexpr int kMaxInternalOrder = 32;  // reference coefficients.hpp:33

// ---------------------------------------------------------------------------
// Hyperspherical harmonics.
std::size_t harmonicIndexCount(int d, int k);
double additionNormalizer(int d, int k);
double gegenbauerAtOne(int d, int k);

struct HarmonicChain {
  std::vector<int> m;  // m[0] = degree, m[1..d-2] >= 0 (absolute values)
  int phase = 0;       // +1 cos, -1 sin, 0 when the last entry is 0
  double norm = 1.0;
};

class HarmonicStructure {
 public:
  HarmonicStructure(int d, int p);
  int dimension() const { return d_; }
  int maxDegree() const { return p_; }
  std::size_t total() const { return total_; }
  std::size_t degreeOffset(int k) const { return offset_[static_cast<std::size_t>(k)]; }
  std::size_t degreeCount(int k) const { return offset_[static_cast<std::size_t>(k) + 1] - offset_[static_cast<std::size_t>(k)]; }
  double z(int k) const { return z_[static_cast<std::size_t>(k)]; }
  const std::vector<HarmonicChain>& chains(int k) const { return chains_[static_cast<std::size_t>(k)]; }

 private:
  int d_, p_;
  std::size_t total_ = 0;
  std::vector<std::size_t> offset_;
  std::vector<double> z_;
  std::vector<std::vector<HarmonicChain>> chains_;
};

// ---------------------------------------------------------------------------
// Exact radial compression.
struct RadialFactor {
  int degree = 0;
  int rank = 0;
  std::vector<Laurent> target;  // multiplies K(r)
  std::vector<Laurent> source;  // polynomials in r'
};

class NotRecurrenceKernelError : public std::invalid_argument {
 public:
  explicit NotRecurrenceKernelError(const std::string& name)
      : std::invalid_argument("kernel '" + name + "' has no registered derivative recurrence") {}
};

std::vector<RadialFactor> radialCompression(const KernelSpec& k, const CoefTable& table, int p);

std::size_t expansionSize(int d, int p);

}  // namespace fktb

#endif
