// Product plan-time exact arithmetic (host only): arbitrary-precision
// integers and normalised rationals for the coefficient tables T-bar
// (reference proj/src/coefficients.cpp:12-111), harmonic counts
// (harmonics.cpp:55-60) and the exact rank-revealing radial compression
// (expansion.cpp:116-243). Same representation as the oracle's Boost shim
// (base-2^32 limbs, Knuth D division, round-to-nearest-even conversion), kept
// as a separate product copy so nothing in the product links oracle/.
#ifndef FKTB_EXACT_HPP
#define FKTB_EXACT_HPP

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace fktb {
namespace exact {

class BigInt {
 public:
  using limb = std::uint32_t;

  BigInt() = default;
  template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
  BigInt(I v) {  // NOLINT(implicit)
    if constexpr (std::is_signed_v<I>) {
      if (v < 0) {
        neg_ = true;
        setMag(static_cast<unsigned long long>(-(static_cast<long long>(v) + 1)) + 1ull);
        return;
      }
    }
    setMag(static_cast<unsigned long long>(v));
  }

  bool isZero() const { return mag_.empty(); }
  bool negative() const { return neg_; }
  const std::vector<limb>& mag() const { return mag_; }

  template <class T>
  T convert_to() const {
    if constexpr (std::is_floating_point_v<T>) {
      // Exact enough for the reference's uses (binomials); correctly rounded
      // via the rational path is not needed for integers below 2^53.
      long double acc = 0;
      for (std::size_t i = mag_.size(); i-- > 0;) acc = acc * 4294967296.0L + mag_[i];
      return static_cast<T>(neg_ ? -acc : acc);
    } else {
      unsigned long long v = 0;
      for (std::size_t i = std::min<std::size_t>(mag_.size(), 2); i-- > 0;) v = (v << 32) | mag_[i];
      if (neg_) return static_cast<T>(-static_cast<long long>(v));
      return static_cast<T>(v);
    }
  }

  friend BigInt operator-(BigInt a) {
    if (!a.isZero()) a.neg_ = !a.neg_;
    return a;
  }
  friend BigInt operator+(const BigInt& a, const BigInt& b) {
    if (a.neg_ == b.neg_) return make(addMag(a.mag_, b.mag_), a.neg_);
    const int c = cmpMag(a.mag_, b.mag_);
    if (c == 0) return BigInt();
    if (c > 0) return make(subMag(a.mag_, b.mag_), a.neg_);
    return make(subMag(b.mag_, a.mag_), b.neg_);
  }
  friend BigInt operator-(const BigInt& a, const BigInt& b) { return a + (-b); }
  friend BigInt operator*(const BigInt& a, const BigInt& b) {
    return make(mulMag(a.mag_, b.mag_), a.neg_ != b.neg_);
  }
  // Truncating division, like C++ integers and Boost.
  friend BigInt operator/(const BigInt& a, const BigInt& b) {
    std::vector<limb> q, r;
    divMag(a.mag_, b.mag_, q, r);
    return make(std::move(q), a.neg_ != b.neg_);
  }
  friend BigInt operator%(const BigInt& a, const BigInt& b) {
    std::vector<limb> q, r;
    divMag(a.mag_, b.mag_, q, r);
    return make(std::move(r), a.neg_);
  }
  BigInt& operator+=(const BigInt& o) { return *this = *this + o; }
  BigInt& operator-=(const BigInt& o) { return *this = *this - o; }
  BigInt& operator*=(const BigInt& o) { return *this = *this * o; }
  BigInt& operator/=(const BigInt& o) { return *this = *this / o; }
  BigInt& operator%=(const BigInt& o) { return *this = *this % o; }

  friend BigInt operator<<(const BigInt& a, unsigned s) { return make(shlMag(a.mag_, s), a.neg_); }
  friend BigInt operator>>(const BigInt& a, unsigned s) { return make(shrMag(a.mag_, s), a.neg_); }

  friend int compare(const BigInt& a, const BigInt& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    const int c = cmpMag(a.mag_, b.mag_);
    return a.neg_ ? -c : c;
  }
  friend bool operator==(const BigInt& a, const BigInt& b) { return a.neg_ == b.neg_ && a.mag_ == b.mag_; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return !(a == b); }
  friend bool operator<(const BigInt& a, const BigInt& b) { return compare(a, b) < 0; }
  friend bool operator>(const BigInt& a, const BigInt& b) { return compare(a, b) > 0; }
  friend bool operator<=(const BigInt& a, const BigInt& b) { return compare(a, b) <= 0; }
  friend bool operator>=(const BigInt& a, const BigInt& b) { return compare(a, b) >= 0; }

  std::size_t bitLength() const {
    if (mag_.empty()) return 0;
    std::size_t b = 32 * (mag_.size() - 1);
    limb top = mag_.back();
    while (top) {
      ++b;
      top >>= 1;
    }
    return b;
  }
  bool bit(std::size_t i) const {
    const std::size_t w = i / 32;
    return w < mag_.size() && ((mag_[w] >> (i % 32)) & 1u);
  }

  std::string str() const {
    if (mag_.empty()) return "0";
    std::vector<limb> cur = mag_;
    std::string digits;
    while (!cur.empty()) {
      // divide by 1e9
      unsigned long long rem = 0;
      for (std::size_t i = cur.size(); i-- > 0;) {
        const unsigned long long v = (rem << 32) | cur[i];
        cur[i] = static_cast<limb>(v / 1000000000ull);
        rem = v % 1000000000ull;
      }
      trim(cur);
      for (int k = 0; k < 9; ++k) {
        digits.push_back(static_cast<char>('0' + rem % 10));
        rem /= 10;
        if (cur.empty() && rem == 0) break;
      }
    }
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    if (neg_) digits.push_back('-');
    std::reverse(digits.begin(), digits.end());
    return digits;
  }

  friend std::ostream& operator<<(std::ostream& os, const BigInt& v) { return os << v.str(); }
  friend std::istream& operator>>(std::istream& is, BigInt& v) {
    std::string s;
    if (!(is >> s)) return is;
    std::size_t i = 0;
    bool neg = false;
    if (i < s.size() && (s[i] == '-' || s[i] == '+')) {
      neg = s[i] == '-';
      ++i;
    }
    if (i == s.size()) {
      is.setstate(std::ios::failbit);
      return is;
    }
    BigInt acc;
    for (; i < s.size(); ++i) {
      if (s[i] < '0' || s[i] > '9') {
        is.setstate(std::ios::failbit);
        return is;
      }
      acc = acc * BigInt(10) + BigInt(s[i] - '0');
    }
    v = neg ? -acc : acc;
    return is;
  }

  static BigInt make(std::vector<limb> m, bool neg) {
    BigInt r;
    trim(m);
    r.mag_ = std::move(m);
    r.neg_ = neg && !r.mag_.empty();
    return r;
  }

 private:
  void setMag(unsigned long long v) {
    mag_.clear();
    while (v) {
      mag_.push_back(static_cast<limb>(v & 0xffffffffull));
      v >>= 32;
    }
  }
  static void trim(std::vector<limb>& m) {
    while (!m.empty() && m.back() == 0) m.pop_back();
  }
  static int cmpMag(const std::vector<limb>& a, const std::vector<limb>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static std::vector<limb> addMag(const std::vector<limb>& a, const std::vector<limb>& b) {
    std::vector<limb> r(std::max(a.size(), b.size()) + 1, 0);
    unsigned long long carry = 0;
    for (std::size_t i = 0; i < r.size(); ++i) {
      unsigned long long s = carry;
      if (i < a.size()) s += a[i];
      if (i < b.size()) s += b[i];
      r[i] = static_cast<limb>(s);
      carry = s >> 32;
    }
    trim(r);
    return r;
  }
  // requires |a| >= |b|
  static std::vector<limb> subMag(const std::vector<limb>& a, const std::vector<limb>& b) {
    std::vector<limb> r(a.size(), 0);
    long long borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      long long s = static_cast<long long>(a[i]) - borrow - (i < b.size() ? static_cast<long long>(b[i]) : 0);
      borrow = 0;
      if (s < 0) {
        s += 4294967296ll;
        borrow = 1;
      }
      r[i] = static_cast<limb>(s);
    }
    trim(r);
    return r;
  }
  static std::vector<limb> mulMag(const std::vector<limb>& a, const std::vector<limb>& b) {
    if (a.empty() || b.empty()) return {};
    std::vector<limb> r(a.size() + b.size(), 0);
    for (std::size_t i = 0; i < a.size(); ++i) {
      unsigned long long carry = 0;
      for (std::size_t j = 0; j < b.size(); ++j) {
        const unsigned long long t = static_cast<unsigned long long>(a[i]) * b[j] + r[i + j] + carry;
        r[i + j] = static_cast<limb>(t);
        carry = t >> 32;
      }
      std::size_t k = i + b.size();
      while (carry) {
        const unsigned long long t = static_cast<unsigned long long>(r[k]) + carry;
        r[k] = static_cast<limb>(t);
        carry = t >> 32;
        ++k;
      }
    }
    trim(r);
    return r;
  }
  static std::vector<limb> shlMag(const std::vector<limb>& a, unsigned s) {
    if (a.empty()) return {};
    const unsigned w = s / 32, b = s % 32;
    std::vector<limb> r(a.size() + w + 1, 0);
    for (std::size_t i = 0; i < a.size(); ++i) {
      const unsigned long long v = static_cast<unsigned long long>(a[i]) << b;
      r[i + w] |= static_cast<limb>(v);
      r[i + w + 1] |= static_cast<limb>(v >> 32);
    }
    trim(r);
    return r;
  }
  static std::vector<limb> shrMag(const std::vector<limb>& a, unsigned s) {
    const unsigned w = s / 32, b = s % 32;
    if (w >= a.size()) return {};
    std::vector<limb> r(a.size() - w, 0);
    for (std::size_t i = 0; i < r.size(); ++i) {
      unsigned long long v = a[i + w];
      if (i + w + 1 < a.size()) v |= static_cast<unsigned long long>(a[i + w + 1]) << 32;
      r[i] = static_cast<limb>(v >> b);
    }
    trim(r);
    return r;
  }
  // Knuth, TAOCP vol. 2, 4.3.1 Algorithm D (schoolbook long division).
  static void divMag(const std::vector<limb>& a, const std::vector<limb>& b, std::vector<limb>& q,
                     std::vector<limb>& r) {
    if (b.empty()) throw std::domain_error("BigInt: division by zero");
    if (cmpMag(a, b) < 0) {
      q.clear();
      r = a;
      return;
    }
    if (b.size() == 1) {
      q.assign(a.size(), 0);
      unsigned long long rem = 0;
      for (std::size_t i = a.size(); i-- > 0;) {
        const unsigned long long v = (rem << 32) | a[i];
        q[i] = static_cast<limb>(v / b[0]);
        rem = v % b[0];
      }
      trim(q);
      r.clear();
      if (rem) r.push_back(static_cast<limb>(rem));
      return;
    }
    unsigned s = 0;
    while (((b.back() << s) & 0x80000000u) == 0) ++s;
    std::vector<limb> v = shlMag(b, s);
    std::vector<limb> u = shlMag(a, s);
    u.resize(a.size() + 1, 0);
    if (u.size() < a.size() + 1) u.resize(a.size() + 1, 0);
    const std::size_t n = v.size(), m = u.size() - n;
    q.assign(m, 0);
    const unsigned long long B = 4294967296ull;
    for (std::size_t jj = m; jj-- > 0;) {
      const unsigned long long num = (static_cast<unsigned long long>(u[jj + n]) << 32) | u[jj + n - 1];
      unsigned long long qhat = num / v[n - 1];
      unsigned long long rhat = num % v[n - 1];
      while (qhat >= B || qhat * v[n - 2] > ((rhat << 32) | u[jj + n - 2])) {
        --qhat;
        rhat += v[n - 1];
        if (rhat >= B) break;
      }
      long long borrow = 0;
      unsigned long long carry = 0;
      for (std::size_t i = 0; i < n; ++i) {
        const unsigned long long p = qhat * v[i] + carry;
        carry = p >> 32;
        long long t = static_cast<long long>(u[i + jj]) - borrow - static_cast<long long>(p & 0xffffffffull);
        borrow = 0;
        if (t < 0) {
          t += static_cast<long long>(B);
          borrow = 1;
        }
        u[i + jj] = static_cast<limb>(t);
      }
      long long t = static_cast<long long>(u[jj + n]) - borrow - static_cast<long long>(carry);
      borrow = 0;
      if (t < 0) {
        t += static_cast<long long>(B);
        borrow = 1;
      }
      u[jj + n] = static_cast<limb>(t);
      if (borrow) {
        --qhat;
        unsigned long long c = 0;
        for (std::size_t i = 0; i < n; ++i) {
          const unsigned long long s2 = static_cast<unsigned long long>(u[i + jj]) + v[i] + c;
          u[i + jj] = static_cast<limb>(s2);
          c = s2 >> 32;
        }
        u[jj + n] = static_cast<limb>(static_cast<unsigned long long>(u[jj + n]) + c);
      }
      q[jj] = static_cast<limb>(qhat);
    }
    trim(q);
    u.resize(n);
    trim(u);
    r = shrMag(u, s);
  }

  bool neg_ = false;
  std::vector<limb> mag_;
};

inline BigInt abs(const BigInt& a) { return a.negative() ? -a : a; }

inline BigInt gcd(BigInt a, BigInt b) {
  a = abs(a);
  b = abs(b);
  while (!b.isZero()) {
    BigInt t = a % b;
    a = std::move(b);
    b = std::move(t);
  }
  return a;
}

class Rational {
 public:
  Rational() : num_(0), den_(1) {}
  template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
  Rational(I v) : num_(v), den_(1) {}  // NOLINT(implicit)
  Rational(const BigInt& v) : num_(v), den_(1) {}  // NOLINT(implicit)
  Rational(const BigInt& n, const BigInt& d) : num_(n), den_(d) { normalize(); }
  template <class I, class J, class = std::enable_if_t<std::is_integral_v<I> && std::is_integral_v<J>>>
  Rational(I n, J d) : num_(n), den_(d) {
    normalize();
  }
  // Exact: every finite double is a dyadic rational.
  explicit Rational(double x) : num_(0), den_(1) {
    if (!std::isfinite(x)) throw std::domain_error("Rational: non-finite double");
    if (x == 0.0) return;
    int e = 0;
    const double m = std::frexp(std::fabs(x), &e);  // x = m * 2^e, m in [0.5, 1)
    const long long mant = static_cast<long long>(std::ldexp(m, 53));
    e -= 53;
    num_ = BigInt(mant);
    if (e >= 0)
      num_ = num_ << static_cast<unsigned>(e);
    else
      den_ = BigInt(1) << static_cast<unsigned>(-e);
    if (x < 0) num_ = -num_;
    normalize();
  }

  const BigInt& num() const { return num_; }
  const BigInt& den() const { return den_; }

  template <class T>
  T convert_to() const {
    static_assert(std::is_floating_point_v<T>, "Rational::convert_to supports floating types");
    return static_cast<T>(toDoubleRounded());
  }

  friend Rational operator-(Rational a) {
    a.num_ = -a.num_;
    return a;
  }
  friend Rational operator+(const Rational& a, const Rational& b) {
    return Rational(a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_);
  }
  friend Rational operator-(const Rational& a, const Rational& b) {
    return Rational(a.num_ * b.den_ - b.num_ * a.den_, a.den_ * b.den_);
  }
  friend Rational operator*(const Rational& a, const Rational& b) {
    return Rational(a.num_ * b.num_, a.den_ * b.den_);
  }
  friend Rational operator/(const Rational& a, const Rational& b) {
    if (b.num_.isZero()) throw std::domain_error("Rational: division by zero");
    return Rational(a.num_ * b.den_, a.den_ * b.num_);
  }
  Rational& operator+=(const Rational& o) { return *this = *this + o; }
  Rational& operator-=(const Rational& o) { return *this = *this - o; }
  Rational& operator*=(const Rational& o) { return *this = *this * o; }
  Rational& operator/=(const Rational& o) { return *this = *this / o; }

  friend bool operator==(const Rational& a, const Rational& b) { return a.num_ == b.num_ && a.den_ == b.den_; }
  friend bool operator!=(const Rational& a, const Rational& b) { return !(a == b); }
  friend bool operator<(const Rational& a, const Rational& b) { return a.num_ * b.den_ < b.num_ * a.den_; }
  friend bool operator>(const Rational& a, const Rational& b) { return b < a; }
  friend bool operator<=(const Rational& a, const Rational& b) { return !(b < a); }
  friend bool operator>=(const Rational& a, const Rational& b) { return !(a < b); }

  friend std::ostream& operator<<(std::ostream& os, const Rational& q) {
    os << q.num_;
    if (q.den_ != BigInt(1)) os << "/" << q.den_;
    return os;
  }

 private:
  void normalize() {
    if (den_.isZero()) throw std::domain_error("Rational: zero denominator");
    if (den_.negative()) {
      num_ = -num_;
      den_ = -den_;
    }
    if (num_.isZero()) {
      den_ = BigInt(1);
      return;
    }
    const BigInt g = gcd(num_, den_);
    if (g != BigInt(1)) {
      num_ = num_ / g;
      den_ = den_ / g;
    }
  }

  // Round-to-nearest-even of num/den (normal range).
  double toDoubleRounded() const {
    if (num_.isZero()) return 0.0;
    const bool neg = num_.negative();
    const BigInt a = abs(num_);
    const long long la = static_cast<long long>(a.bitLength());
    const long long lb = static_cast<long long>(den_.bitLength());
    // Scale so the integer quotient has 55..56 bits (53 + guard + sticky room).
    long long shift = 55 - (la - lb);
    BigInt n = a, d = den_;
    if (shift >= 0)
      n = n << static_cast<unsigned>(shift);
    else
      d = d << static_cast<unsigned>(-shift);
    BigInt q = n / d;
    const bool sticky0 = !(n % d).isZero();
    // Reduce q to exactly 54 bits (53 + round bit), folding lost bits into sticky.
    long long qb = static_cast<long long>(q.bitLength());
    bool sticky = sticky0;
    long long extra = qb - 54;
    if (extra > 0) {
      for (long long i = 0; i < extra; ++i)
        if (q.bit(static_cast<std::size_t>(i))) sticky = true;
      q = q >> static_cast<unsigned>(extra);
      shift -= extra;
    }
    unsigned long long m = q.convert_to<unsigned long long>();
    const bool roundBit = m & 1ull;
    m >>= 1;
    shift -= 1;
    if (roundBit && (sticky || (m & 1ull))) {
      ++m;
      if (m == (1ull << 53)) {
        m >>= 1;
        shift -= 1;
      }
    }
    double r = std::ldexp(static_cast<double>(m), static_cast<int>(-shift));
    return neg ? -r : r;
  }

  BigInt num_, den_;
};

inline const BigInt& numerator(const Rational& q) { return q.num(); }
inline const BigInt& denominator(const Rational& q) { return q.den(); }

}  // namespace exact
}  // namespace fktb

#endif
