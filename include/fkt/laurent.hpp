// B200-native FKT — C++ operator API: exact rational Laurent polynomials for
// the kernels' registered derivative recurrences K'(r) = q(r) K(r) (the role
// of the reference's RationalLaurent, proj/include/fkt/laurent.hpp). The
// coefficients are exact rationals carried as decimal numerator / denominator
// strings (parameters enter as the exact dyadic rationals of their doubles),
// so nothing is rounded on the way from the library to the caller.
#ifndef FKT_B200_LAURENT_HPP
#define FKT_B200_LAURENT_HPP

#include <cmath>
#include <cstdlib>
#include <map>
#include <string>

namespace fkt {

struct ExactRational {
  std::string numerator = "0", denominator = "1";
  bool operator==(const ExactRational& o) const { return numerator == o.numerator && denominator == o.denominator; }
  bool operator!=(const ExactRational& o) const { return !(*this == o); }
  // nearest double (long double division of the parsed integers)
  double toDouble() const { return static_cast<double>(std::strtold(numerator.c_str(), nullptr) /
                                                       std::strtold(denominator.c_str(), nullptr)); }
};

class RationalLaurent {
 public:
  void add(int power, ExactRational c) {
    if (c.numerator != "0") terms_[power] = std::move(c);
  }
  ExactRational coeff(int power) const {
    auto it = terms_.find(power);
    return it == terms_.end() ? ExactRational{} : it->second;
  }
  bool empty() const { return terms_.empty(); }
  int minPower() const { return terms_.empty() ? 0 : terms_.begin()->first; }
  int maxPower() const { return terms_.empty() ? 0 : terms_.rbegin()->first; }
  const std::map<int, ExactRational>& terms() const { return terms_; }
  // q(r) in double precision, r != 0 when a negative power is present
  double operator()(double r) const {
    double s = 0.0;
    for (const auto& [p, c] : terms_) s += c.toDouble() * std::pow(r, p);
    return s;
  }
  bool operator==(const RationalLaurent& o) const { return terms_ == o.terms_; }

 private:
  std::map<int, ExactRational> terms_;
};

}  // namespace fkt

#endif
