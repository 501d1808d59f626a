// B200-native FKT — seeded synthetic inputs (drop-in for the reference's
// proj/include/fkt/synthetic.hpp:17-62). Same streams as the reference:
// splitmix64 increments, 53-bit uniforms, Box-Muller normals that cache the
// sine branch for the next call. Implemented in cpp/fkt_api.cpp.
#ifndef FKT_B200_SYNTHETIC_HPP
#define FKT_B200_SYNTHETIC_HPP

#include <cstdint>
#include <vector>

#include "fkt/tree.hpp"

namespace fkt {

class Rng {
 public:
  explicit Rng(std::uint64_t seed);
  std::uint64_t next();
  double uniform();
  double uniform(double lo, double hi);
  double normal();

 private:
  std::uint64_t s_;
  double cached_ = 0.0;
  bool cachedValid_ = false;
};

PointCloud sphereSurfaceCloud(int n, int d, Rng& rng);
PointCloud cubeCloud(int n, int d, Rng& rng);
PointCloud gaussianMixtureCloud(int n, int d, Rng& rng, int components = 5);
std::vector<double> normalVector(int n, Rng& rng);

}  // namespace fkt

#endif
