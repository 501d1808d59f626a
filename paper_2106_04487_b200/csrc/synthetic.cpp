// Seeded synthetic inputs: the reference's splitmix64 + Box-Muller RNG
// (proj/include/fkt/synthetic.hpp:17-50) and generators
// (proj/src/synthetic.cpp:7-55), plus the BASELINE config recipes of
// SURVEY Appendix B. Host code; bit-identical inputs to the reference's own
// generator are what make tree/set parity checkable.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace fktb {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state_ += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (haveSpare_) {
      haveSpare_ = false;
      return spare_;
    }
    double u1 = uniform(), u2 = uniform();
    while (u1 <= 1e-300) u1 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 6.283185307179586476925286766559 * u2;
    spare_ = radius * std::sin(angle);
    haveSpare_ = true;
    return radius * std::cos(angle);
  }

 private:
  std::uint64_t state_;
  bool haveSpare_ = false;
  double spare_ = 0.0;
};

void synthCloud(const std::string& kind, int n, int d, std::uint64_t seed, double* x, double* y) {
  Rng rng(seed);
  if (kind == "cube") {
    for (long long i = 0; i < static_cast<long long>(n) * d; ++i) x[i] = rng.uniform();
  } else if (kind == "sphere") {
    for (int i = 0; i < n; ++i) {
      double* pt = x + static_cast<std::size_t>(i) * d;
      double norm2 = 0.0;
      do {
        norm2 = 0.0;
        for (int a = 0; a < d; ++a) {
          pt[a] = rng.normal();
          norm2 += pt[a] * pt[a];
        }
      } while (norm2 == 0.0);
      const double inv = 1.0 / std::sqrt(norm2);
      for (int a = 0; a < d; ++a) pt[a] *= inv;
    }
  } else if (kind == "mixture") {
    const int components = 5;
    std::vector<double> centers(static_cast<std::size_t>(components) * d), widths(components);
    for (int c = 0; c < components; ++c) {
      for (int a = 0; a < d; ++a) centers[static_cast<std::size_t>(c) * d + a] = rng.uniform(-1.0, 1.0);
      widths[static_cast<std::size_t>(c)] = rng.uniform(0.05, 0.25);
    }
    for (int i = 0; i < n; ++i) {
      const int c = static_cast<int>(rng.next() % static_cast<std::uint64_t>(components));
      for (int a = 0; a < d; ++a)
        x[static_cast<std::size_t>(i) * d + a] = centers[static_cast<std::size_t>(c) * d + a] + widths[static_cast<std::size_t>(c)] * rng.normal();
    }
  } else {
    throw std::invalid_argument("unknown cloud kind '" + kind + "'");
  }
  if (y)
    for (int i = 0; i < n; ++i) y[i] = rng.normal();
}

int configDims(int cfg, int* d, int* nrhs) {
  static const int dims[6] = {0, 3, 3, 5, 3, 2};
  if (cfg < 1 || cfg > 5) return -1;
  *d = dims[cfg];
  *nrhs = cfg == 5 ? 16 : 1;
  return 0;
}

// SURVEY Appendix B (points first, then weights, one Rng stream).
void synthConfig(int cfg, int n, std::uint64_t seed, double* x, double* w) {
  int d = 0, nrhs = 0;
  if (configDims(cfg, &d, &nrhs) != 0) throw std::invalid_argument("config must be 1..5");
  Rng rng(seed);
  const std::size_t nd = static_cast<std::size_t>(n) * d;
  if (cfg == 1 || cfg == 2) {
    for (std::size_t i = 0; i < nd; ++i) x[i] = rng.uniform();
    for (int i = 0; i < n; ++i) w[i] = rng.normal();
  } else if (cfg == 3) {
    double mu[8][5];
    for (auto& row : mu)
      for (double& v : row) v = rng.uniform();
    for (int i = 0; i < n; ++i) {
      const int c = static_cast<int>(rng.next() % 8);
      for (int a = 0; a < 5; ++a) x[static_cast<std::size_t>(i) * 5 + a] = mu[c][a] + 0.05 * rng.normal();
    }
    const double s = std::sqrt(2.0);
    for (std::size_t i = 0; i < nd; ++i) x[i] *= s;
    for (int i = 0; i < n; ++i) w[i] = rng.normal();
  } else if (cfg == 4) {
    for (int i = 0; i < n; ++i) {
      double* pt = x + static_cast<std::size_t>(i) * 3;
      double norm2 = 0.0;
      do {
        norm2 = 0.0;
        for (int a = 0; a < 3; ++a) {
          pt[a] = rng.normal();
          norm2 += pt[a] * pt[a];
        }
      } while (norm2 == 0.0);
      const double inv = 1.0 / std::sqrt(norm2);
      for (int a = 0; a < 3; ++a) pt[a] *= inv;
    }
    for (int i = 0; i < n; ++i) {
      const double s = 1.0 + 0.01 * rng.normal();
      for (int a = 0; a < 3; ++a) x[static_cast<std::size_t>(i) * 3 + a] *= s;
    }
    for (int i = 0; i < n; ++i) w[i] = rng.uniform(-1.0, 1.0);
  } else {
    double mu[10][2];
    for (auto& row : mu)
      for (double& v : row) v = rng.uniform(-50.0, 50.0);
    for (int i = 0; i < n; ++i) {
      const int c = static_cast<int>(rng.next() % 10);
      for (int a = 0; a < 2; ++a) x[static_cast<std::size_t>(i) * 2 + a] = mu[c][a] + 3.0 * rng.normal();
    }
    for (int r = 0; r < 16; ++r)
      for (int i = 0; i < n; ++i) w[static_cast<std::size_t>(r) * n + i] = rng.normal();
  }
}

}  // namespace fktb
