// B200-native FKT — C++ operator API, the transform (drop-in for the
// reference's proj/include/fkt/transform.hpp:15-87). FktPlan builds the tree,
// interaction sets and expansion tables on one GPU; multiply() runs the MVM
// there (host buffers in, host buffers out). Additive extensions: a
// multi-right-hand-side multiply and a device-pointer multiply.
#ifndef FKT_B200_TRANSFORM_HPP
#define FKT_B200_TRANSFORM_HPP

#include <cstddef>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fkt/kernels.hpp"
#include "fkt/tree.hpp"

namespace fkt {

class DimensionMismatchError : public std::invalid_argument {
 public:
  explicit DimensionMismatchError(const std::string& what) : std::invalid_argument(what) {}
};

class ZeroReferenceError : public std::invalid_argument {
 public:
  ZeroReferenceError() : std::invalid_argument("relative error against a zero reference vector") {}
};

class OrderTooLargeError : public std::invalid_argument {
 public:
  explicit OrderTooLargeError(const std::string& what) : std::invalid_argument(what) {}
};

class NotRecurrenceKernelError : public std::invalid_argument {
 public:
  explicit NotRecurrenceKernelError(const std::string& what) : std::invalid_argument(what) {}
};

enum class CompressionMode { Auto, On, Off };

struct FktOptions {
  int p = 4;
  double theta = 0.75;
  int leafCapacity = 512;
  CompressionMode compression = CompressionMode::Auto;
  bool eagerOperators = true;  // accepted; the GPU recomputes operators in registers
  bool barnesHut = false;      // monopole far field about centres of mass (csrc/bh.cu); forces p = 0
  int threads = 0;             // CPU knob of the reference, ignored
  std::optional<double> diagonal;
  int nearPrecision = 64;      // additive: 32 selects the FP32 fast near field
  bool deterministic = false;  // additive: bitwise reproducible z (no atomics into z / moments)
};

class FktPlan {
 public:
  FktPlan(PointCloud cloud, KernelPtr kernel, const FktOptions& options);
  ~FktPlan();
  FktPlan(FktPlan&&) noexcept;
  FktPlan& operator=(FktPlan&&) noexcept;
  FktPlan(const FktPlan&) = delete;
  FktPlan& operator=(const FktPlan&) = delete;

  std::vector<double> multiply(std::span<const double> y) const;
  // nrhs column-major right-hand sides (y.size() == n * nrhs).
  std::vector<double> multiply(std::span<const double> y, int nrhs) const;
  // Device buffers (n * nrhs doubles each) on a cudaStream_t (nullptr: the
  // plan's own stream, synchronised before return).
  void multiplyDevice(const double* yDevice, double* zDevice, int nrhs = 1, void* stream = nullptr) const;
  // Additive: the same plan on new coordinates of the same n points (moving
  // points); equals FktPlan(cloud, kernel(), options()), reusing the plan's
  // device buffers. DimensionMismatchError on a different n or d.
  void rebuild(PointCloud cloud);

  const PointCloud& cloud() const { return cloud_; }
  const PartitionTree& tree() const;
  const IsotropicKernel& kernel() const { return *kernel_; }
  const FktOptions& options() const { return options_; }
  bool compressed() const;
  std::size_t coefficientCount() const;
  double planSeconds() const;

  void* handle() const { return h_; }

 private:
  PointCloud cloud_;
  KernelPtr kernel_;
  FktOptions options_;
  void* h_ = nullptr;
  mutable std::unique_ptr<PartitionTree> tree_;
};

FktPlan plan(const PointCloud& cloud, KernelPtr kernel, const FktOptions& options = {});

std::vector<double> denseMultiply(const PointCloud& cloud, const IsotropicKernel& kernel, std::span<const double> y,
                                  std::optional<double> diagonal = std::nullopt, int threads = 0);

std::vector<double> barnesHutMultiply(const FktPlan& plan, std::span<const double> y);

double relativeError(std::span<const double> approx, std::span<const double> exact);

std::size_t expansionSize(int d, int p);

}  // namespace fkt

#endif
