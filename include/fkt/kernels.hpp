// B200-native FKT — C++ operator API, kernels (drop-in for the reference's
// proj/include/fkt/kernels.hpp:22-89). Built-in kernels are identified by
// name + parameters and evaluated on the GPU; kernels built from arbitrary
// host lambdas cannot run there and are rejected by FktPlan.
#ifndef FKT_B200_KERNELS_HPP
#define FKT_B200_KERNELS_HPP

#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "fkt/jet.hpp"
#include "fkt/laurent.hpp"

namespace fkt {

class SingularAtZeroError : public std::domain_error {
 public:
  explicit SingularAtZeroError(const std::string& name)
      : std::domain_error("kernel '" + name + "' is singular at r = 0 and no diagonal convention is set") {}
};

// A valid reference input the GPU path does not offer (there is no CPU fallback).
class UnsupportedOnGpuError : public std::invalid_argument {
 public:
  explicit UnsupportedOnGpuError(const std::string& what) : std::invalid_argument(what) {}
};

class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& what) : std::runtime_error(what) {}
};

class IsotropicKernel {
 public:
  using Params = std::map<std::string, double>;

  // Built-in kernel (see makeKernel).
  IsotropicKernel(std::string name, Params params);
  // Custom host kernel: usable for host evaluation only (FktPlan throws
  // UnsupportedOnGpuError). Mirrors the reference constructor's evaluator /
  // value-at-zero arguments (kernels.hpp:32-42).
  IsotropicKernel(std::string name, Params params, std::function<double(double)> eval,
                  std::optional<double> valueAtZero);
  // The reference's full constructor (kernels.hpp:32-42): evaluator, jet
  // evaluator, registered recurrence, value at zero (host-only, as above).
  IsotropicKernel(std::string name, Params params, std::function<double(double)> eval,
                  std::function<Jet(const Jet&)> evalJet, std::optional<RationalLaurent> recurrence,
                  std::optional<double> valueAtZero);

  const std::string& name() const { return name_; }
  const Params& parameters() const { return params_; }
  bool builtin() const { return builtin_; }

  // K(r) for r > 0; at r = 0 the override, else the convention, else throw.
  double operator()(double r, std::optional<double> diagonalOverride = std::nullopt) const;
  double evalPositive(double r) const;
  bool hasDerivativeRecurrence() const { return recurrence_; }
  std::optional<double> valueAtZero() const { return valueAtZero_; }
  // Jet of K at r > 0: coefficient m is K^(m)(r) / m! (kernels.hpp:61-64).
  Jet jetAt(double r, int order) const;
  // K on a jet argument (kernels.hpp:66).
  Jet evalJet(const Jet& r) const;
  // The registered recurrence K' = q K with exact rational q (kernels.hpp:68).
  const std::optional<RationalLaurent>& derivativeRecurrence() const { return recurrenceQ_; }

 private:
  std::string name_;
  Params params_;
  bool builtin_ = true;
  bool recurrence_ = false;
  std::optional<double> valueAtZero_;
  std::function<double(double)> eval_;
  std::function<Jet(const Jet&)> evalJet_;
  std::optional<RationalLaurent> recurrenceQ_;
};

using KernelPtr = std::shared_ptr<const IsotropicKernel>;

// The 14 built-in kernels (reference kernels.cpp:37-156). Unknown names or
// parameters throw std::invalid_argument.
KernelPtr makeKernel(const std::string& name, const IsotropicKernel::Params& params = {});
std::vector<std::string> builtinKernelNames();

// Registered derivative recurrence, if any (kernels.hpp:89).
std::optional<RationalLaurent> detectDerivativeRecurrence(const IsotropicKernel& kernel);

}  // namespace fkt

#endif
