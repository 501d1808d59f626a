// C++ operator API (include/fkt/*.hpp) over the C-ABI (include/fkt_cuda.h).
// Status codes from the C-ABI are rethrown as the reference's exception types
// (proj/include/fkt/transform.hpp:17-25, kernels.hpp:22-26,
// coefficients.hpp:23-28, expansion.hpp:27-31).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>

#include "fkt/gp.hpp"
#include "fkt/kernels.hpp"
#include "fkt/synthetic.hpp"
#include "fkt/transform.hpp"
#include "fkt/tree.hpp"
#include "fkt_cuda.h"

namespace fkt {
namespace {

[[noreturn]] void rethrow(int code) {
  const std::string msg = fkt_last_error();
  switch (code) {
    case FKT_ERR_DIMENSION_MISMATCH: throw DimensionMismatchError(msg);
    case FKT_ERR_ORDER_TOO_LARGE: throw OrderTooLargeError(msg);
    case FKT_ERR_NOT_RECURRENCE: throw NotRecurrenceKernelError(msg);
    case FKT_ERR_SINGULAR_AT_ZERO: {
      // the C-ABI message is SingularAtZeroError's own text: recover the name
      const size_t q0 = msg.find('\''), q1 = q0 == std::string::npos ? q0 : msg.find('\'', q0 + 1);
      throw SingularAtZeroError(q1 == std::string::npos ? msg : msg.substr(q0 + 1, q1 - q0 - 1));
    }
    case FKT_ERR_ZERO_REFERENCE: throw ZeroReferenceError();
    case FKT_ERR_CUDA: throw CudaError(msg);
    case FKT_ERR_UNSUPPORTED: throw UnsupportedOnGpuError(msg);
    case FKT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw std::runtime_error(msg);
  }
}

void check(int code) {
  if (code != FKT_OK) rethrow(code);
}

struct ParamArrays {
  std::vector<const char*> keys;
  std::vector<double> values;
  explicit ParamArrays(const IsotropicKernel::Params& p) {
    for (const auto& kv : p) {
      keys.push_back(kv.first.c_str());
      values.push_back(kv.second);
    }
  }
  const char* const* k() const { return keys.empty() ? nullptr : keys.data(); }
  const double* v() const { return values.empty() ? nullptr : values.data(); }
  int n() const { return static_cast<int>(keys.size()); }
};

void requireBuiltin(const IsotropicKernel& k) {
  if (!k.builtin())
    throw UnsupportedOnGpuError("kernel '" + k.name() +
                                "' is a host lambda: the GPU path evaluates built-in kernels only");
}

}  // namespace

// ---------------------------------------------------------------------------
IsotropicKernel::IsotropicKernel(std::string name, Params params) : name_(std::move(name)), params_(std::move(params)) {
  ParamArrays pa(params_);
  int rec = 0, hv0 = 0;
  double v0 = 0.0;
  check(fkt_kernel_check(name_.c_str(), pa.k(), pa.v(), pa.n(), &rec, &hv0, &v0));
  recurrence_ = rec != 0;
  if (hv0) valueAtZero_ = v0;
  if (recurrence_) {
    int terms = 0;
    int powers[16];
    std::vector<char> buf(1 << 16);
    check(fkt_kernel_recurrence(name_.c_str(), pa.k(), pa.v(), pa.n(), &terms, powers, 16, buf.data(),
                                static_cast<long long>(buf.size())));
    RationalLaurent q;
    const char* s = buf.data();
    for (int i = 0; i < terms; ++i) {
      const std::string t(s);
      s += t.size() + 1;
      const size_t slash = t.find('/');
      q.add(powers[i], ExactRational{t.substr(0, slash), t.substr(slash + 1)});
    }
    recurrenceQ_ = std::move(q);
  }
}

IsotropicKernel::IsotropicKernel(std::string name, Params params, std::function<double(double)> eval,
                                 std::optional<double> valueAtZero)
    : name_(std::move(name)), params_(std::move(params)), builtin_(false), valueAtZero_(valueAtZero),
      eval_(std::move(eval)) {}

IsotropicKernel::IsotropicKernel(std::string name, Params params, std::function<double(double)> eval,
                                 std::function<Jet(const Jet&)> evalJet, std::optional<RationalLaurent> recurrence,
                                 std::optional<double> valueAtZero)
    : name_(std::move(name)), params_(std::move(params)), builtin_(false), recurrence_(recurrence.has_value()),
      valueAtZero_(valueAtZero), eval_(std::move(eval)), evalJet_(std::move(evalJet)),
      recurrenceQ_(std::move(recurrence)) {}

Jet IsotropicKernel::evalJet(const Jet& r) const {
  if (!builtin_) {
    if (!evalJet_) throw std::invalid_argument("kernel '" + name_ + "' has no jet evaluator");
    return evalJet_(r);
  }
  ParamArrays pa(params_);
  Jet out(r.center(), r.order());
  std::vector<double> o(static_cast<std::size_t>(r.order()) + 1);
  check(fkt_kernel_eval_jet(name_.c_str(), pa.k(), pa.v(), pa.n(), r.center(), r.order(), r.coefficients().data(),
                            o.data()));
  for (int i = 0; i <= r.order(); ++i) out.coeff(i) = o[static_cast<std::size_t>(i)];
  return out;
}

Jet IsotropicKernel::jetAt(double r, int order) const {
  if (r <= 0.0) throw std::invalid_argument("kernel jet requires r > 0");
  return evalJet(Jet::variable(r, order));
}

std::optional<RationalLaurent> detectDerivativeRecurrence(const IsotropicKernel& kernel) {
  return kernel.derivativeRecurrence();
}

double IsotropicKernel::evalPositive(double r) const {
  if (!builtin_) return eval_(r);
  ParamArrays pa(params_);
  double out = 0.0;
  check(fkt_kernel_eval(name_.c_str(), pa.k(), pa.v(), pa.n(), &r, &out, 1, 0, 0.0));
  return out;
}

double IsotropicKernel::operator()(double r, std::optional<double> diagonalOverride) const {
  if (r == 0.0) {
    if (diagonalOverride) return *diagonalOverride;
    if (valueAtZero_) return *valueAtZero_;
    throw SingularAtZeroError(name_);
  }
  return evalPositive(r);
}

KernelPtr makeKernel(const std::string& name, const IsotropicKernel::Params& params) {
  return std::make_shared<IsotropicKernel>(name, params);
}

std::vector<std::string> builtinKernelNames() {
  std::vector<std::string> out;
  for (int i = 0; i < fkt_kernel_count(); ++i) out.emplace_back(fkt_kernel_name(i));
  return out;
}

// ---------------------------------------------------------------------------
struct PartitionTree::View {
  std::vector<TreeNode> nodes;
  std::vector<std::uint32_t> order;
  std::vector<double> perm;
  bool setsLoaded = false;
  std::mutex mutex;
};

PartitionTree::PartitionTree(const PointCloud& cloud, int leafCapacity) : n_(cloud.n), d_(cloud.d) {
  fkt_tree_t t = nullptr;
  check(fkt_tree_create(cloud.n, cloud.d, cloud.x.data(), leafCapacity, &t));
  h_ = t;
  owned_ = true;
}

PartitionTree::PartitionTree(void* borrowed, int n, int d) : h_(borrowed), owned_(false), n_(n), d_(d) {
  double th = 0.0;
  check(fkt_tree_sizes(static_cast<fkt_tree_t>(h_), nullptr, nullptr, nullptr, nullptr, &th));
  theta_ = th;
}

PartitionTree::~PartitionTree() {
  if (owned_ && h_) fkt_tree_destroy(static_cast<fkt_tree_t>(h_));
}

PartitionTree::PartitionTree(PartitionTree&& o) noexcept
    : h_(o.h_), owned_(o.owned_), n_(o.n_), d_(o.d_), theta_(o.theta_), view_(std::move(o.view_)) {
  o.h_ = nullptr;
  o.owned_ = false;
}

PartitionTree& PartitionTree::operator=(PartitionTree&& o) noexcept {
  if (this != &o) {
    if (owned_ && h_) fkt_tree_destroy(static_cast<fkt_tree_t>(h_));
    h_ = o.h_;
    owned_ = o.owned_;
    n_ = o.n_;
    d_ = o.d_;
    theta_ = o.theta_;
    view_ = std::move(o.view_);
    o.h_ = nullptr;
    o.owned_ = false;
  }
  return *this;
}

void PartitionTree::computeInteractionSets(double theta) {
  check(fkt_tree_compute_sets(static_cast<fkt_tree_t>(h_), theta));
  theta_ = theta;
  view_.reset();
}

std::size_t PartitionTree::nodeCount() const {
  long long nodes = 0;
  check(fkt_tree_sizes(static_cast<fkt_tree_t>(h_), &nodes, nullptr, nullptr, nullptr, nullptr));
  return static_cast<std::size_t>(nodes);
}

int PartitionTree::depth() const {
  long long depth = 0;
  check(fkt_tree_sizes(static_cast<fkt_tree_t>(h_), nullptr, &depth, nullptr, nullptr, nullptr));
  return static_cast<int>(depth);
}

void PartitionTree::materialize() const {
  if (!view_) view_ = std::make_unique<View>();
  View& v = *view_;
  std::lock_guard<std::mutex> lock(v.mutex);
  auto* t = static_cast<fkt_tree_t>(h_);
  if (v.nodes.empty()) {
    const std::size_t nn = nodeCount();
    std::vector<std::uint32_t> b(nn), e(nn);
    std::vector<int> l(nn), r(nn);
    std::vector<double> rad(nn), c(nn * d_), lo(nn * d_), hi(nn * d_);
    check(fkt_tree_nodes(t, b.data(), e.data(), l.data(), r.data(), rad.data(), c.data(), lo.data(), hi.data()));
    v.nodes.resize(nn);
    for (std::size_t i = 0; i < nn; ++i) {
      TreeNode& nd = v.nodes[i];
      nd.begin = b[i];
      nd.end = e[i];
      nd.left = l[i];
      nd.right = r[i];
      nd.radius = rad[i];
      nd.center.assign(c.begin() + static_cast<long>(i * d_), c.begin() + static_cast<long>((i + 1) * d_));
      nd.boxLo.assign(lo.begin() + static_cast<long>(i * d_), lo.begin() + static_cast<long>((i + 1) * d_));
      nd.boxHi.assign(hi.begin() + static_cast<long>(i * d_), hi.begin() + static_cast<long>((i + 1) * d_));
    }
    v.order.resize(static_cast<std::size_t>(n_));
    check(fkt_tree_order(t, v.order.data()));
    v.perm.resize(static_cast<std::size_t>(n_) * d_);
    check(fkt_tree_points(t, v.perm.data()));
  }
  if (!v.setsLoaded && theta_ > 0.0) {
    long long ft = 0, nt = 0;
    check(fkt_tree_sizes(t, nullptr, nullptr, &ft, &nt, nullptr));
    std::vector<long long> fo(v.nodes.size() + 1), no(v.nodes.size() + 1);
    std::vector<std::uint32_t> fi(static_cast<std::size_t>(std::max(1ll, ft))), ni(static_cast<std::size_t>(std::max(1ll, nt)));
    check(fkt_tree_far_sets(t, fo.data(), fi.data()));
    check(fkt_tree_near_sets(t, no.data(), ni.data()));
    for (std::size_t i = 0; i < v.nodes.size(); ++i) {
      v.nodes[i].farSet.assign(fi.begin() + fo[i], fi.begin() + fo[i + 1]);
      v.nodes[i].nearSet.assign(ni.begin() + no[i], ni.begin() + no[i + 1]);
    }
    v.setsLoaded = true;
  }
}

const TreeNode& PartitionTree::node(std::size_t i) const {
  materialize();
  return view_->nodes.at(i);
}

const std::vector<std::uint32_t>& PartitionTree::order() const {
  materialize();
  return view_->order;
}

std::span<const double> PartitionTree::pointAt(std::uint32_t pos) const {
  materialize();
  return {view_->perm.data() + static_cast<std::size_t>(pos) * d_, static_cast<std::size_t>(d_)};
}

// ---------------------------------------------------------------------------
namespace {
fkt_options toC(const FktOptions& f) {
  fkt_options o;
  fkt_default_options(&o);
  o.p = f.p;
  o.theta = f.theta;
  o.leaf_capacity = f.leafCapacity;
  o.compression = f.compression == CompressionMode::On    ? FKT_COMPRESSION_ON
                  : f.compression == CompressionMode::Off ? FKT_COMPRESSION_OFF
                                                          : FKT_COMPRESSION_AUTO;
  o.eager_operators = f.eagerOperators ? 1 : 0;
  o.barnes_hut = f.barnesHut ? 1 : 0;
  o.threads = f.threads;
  o.has_diagonal = f.diagonal ? 1 : 0;
  o.diagonal = f.diagonal.value_or(0.0);
  o.near_precision = f.nearPrecision;
  o.deterministic = f.deterministic ? 1 : 0;
  return o;
}
}  // namespace

FktPlan::FktPlan(PointCloud cloud, KernelPtr kernel, const FktOptions& options)
    : cloud_(std::move(cloud)), kernel_(std::move(kernel)), options_(options) {
  requireBuiltin(*kernel_);
  const fkt_options o = toC(options_);
  ParamArrays pa(kernel_->parameters());
  fkt_plan_t h = nullptr;
  check(fkt_plan_create(cloud_.n, cloud_.d, cloud_.x.data(), kernel_->name().c_str(), pa.k(), pa.v(), pa.n(), &o, &h));
  h_ = h;
  if (options_.barnesHut) options_.p = 0;  // transform.cpp:44
}

FktPlan::~FktPlan() {
  tree_.reset();
  if (h_) fkt_plan_destroy(static_cast<fkt_plan_t>(h_));
}

FktPlan::FktPlan(FktPlan&& o) noexcept
    : cloud_(std::move(o.cloud_)), kernel_(std::move(o.kernel_)), options_(o.options_), h_(o.h_),
      tree_(std::move(o.tree_)) {
  o.h_ = nullptr;
}

FktPlan& FktPlan::operator=(FktPlan&& o) noexcept {
  if (this != &o) {
    tree_.reset();
    if (h_) fkt_plan_destroy(static_cast<fkt_plan_t>(h_));
    cloud_ = std::move(o.cloud_);
    kernel_ = std::move(o.kernel_);
    options_ = o.options_;
    h_ = o.h_;
    tree_ = std::move(o.tree_);
    o.h_ = nullptr;
  }
  return *this;
}

std::vector<double> FktPlan::multiply(std::span<const double> y) const { return multiply(y, 1); }

std::vector<double> FktPlan::multiply(std::span<const double> y, int nrhs) const {
  if (nrhs < 1 || y.size() != static_cast<std::size_t>(cloud_.n) * static_cast<std::size_t>(nrhs))
    throw DimensionMismatchError("multiply: vector length does not match the point count");
  std::vector<double> z(y.size());
  check(fkt_plan_multiply(static_cast<fkt_plan_t>(h_), y.data(), z.data(), nrhs));
  return z;
}

void FktPlan::rebuild(PointCloud cloud) {
  if (cloud.n != cloud_.n || cloud.d != cloud_.d)
    throw DimensionMismatchError("rebuild: the cloud must have the plan's n points in d dimensions");
  check(fkt_plan_rebuild(static_cast<fkt_plan_t>(h_), cloud.x.data()));
  cloud_ = std::move(cloud);
  tree_.reset();
}

void FktPlan::multiplyDevice(const double* y, double* z, int nrhs, void* stream) const {
  check(fkt_plan_multiply_device(static_cast<fkt_plan_t>(h_), y, z, nrhs, stream));
}

const PartitionTree& FktPlan::tree() const {
  if (!tree_) tree_.reset(new PartitionTree(fkt_plan_tree(static_cast<fkt_plan_t>(h_)), cloud_.n, cloud_.d));
  return *tree_;
}

bool FktPlan::compressed() const {
  fkt_plan_info info;
  check(fkt_plan_info_get(static_cast<fkt_plan_t>(h_), &info));
  return info.compressed != 0;
}

std::size_t FktPlan::coefficientCount() const {
  fkt_plan_info info;
  check(fkt_plan_info_get(static_cast<fkt_plan_t>(h_), &info));
  return static_cast<std::size_t>(info.coefficient_count);
}

double FktPlan::planSeconds() const {
  fkt_plan_info info;
  check(fkt_plan_info_get(static_cast<fkt_plan_t>(h_), &info));
  return info.plan_seconds;
}

FktPlan plan(const PointCloud& cloud, KernelPtr kernel, const FktOptions& options) {
  return FktPlan(cloud, std::move(kernel), options);
}

std::vector<double> denseMultiply(const PointCloud& cloud, const IsotropicKernel& kernel, std::span<const double> y,
                                  std::optional<double> diagonal, int /*threads*/) {
  if (y.size() != static_cast<std::size_t>(cloud.n))
    throw DimensionMismatchError("denseMultiply: vector length does not match the point count");
  requireBuiltin(kernel);
  ParamArrays pa(kernel.parameters());
  std::vector<double> z(static_cast<std::size_t>(cloud.n));
  check(fkt_dense_multiply(cloud.n, cloud.d, cloud.x.data(), kernel.name().c_str(), pa.k(), pa.v(), pa.n(), y.data(),
                           z.data(), diagonal ? 1 : 0, diagonal.value_or(0.0)));
  return z;
}

std::vector<double> barnesHutMultiply(const FktPlan& plan, std::span<const double> y) {
  if (!plan.options().barnesHut)
    throw std::invalid_argument("barnesHutMultiply requires a plan built with the Barnes-Hut option");
  return plan.multiply(y);
}

double relativeError(std::span<const double> approx, std::span<const double> exact) {
  if (approx.size() != exact.size()) throw DimensionMismatchError("relativeError: length mismatch");
  double out = 0.0;
  check(fkt_relative_error(approx.data(), exact.data(), static_cast<long long>(approx.size()), &out));
  return out;
}

std::size_t expansionSize(int d, int p) {
  const long long r = fkt_expansion_size(d, p);
  if (r < 0) rethrow(fkt_last_error_code());
  return static_cast<std::size_t>(r);
}

// ---------------------------------------------------------------------------
// Seeded inputs: splitmix64 stream, 53-bit uniforms, Box-Muller with the sine
// branch cached (same streams as proj/include/fkt/synthetic.hpp:17-50).
namespace {
constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
}  // namespace

Rng::Rng(std::uint64_t seed) : s_(seed) {}

std::uint64_t Rng::next() {
  s_ += kGolden;
  return mix64(s_);
}

double Rng::uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

double Rng::uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

double Rng::normal() {
  if (cachedValid_) {
    cachedValid_ = false;
    return cached_;
  }
  double a = uniform();
  const double b = uniform();
  while (a <= 1e-300) a = uniform();
  const double rad = std::sqrt(-2.0 * std::log(a));
  const double ang = 6.283185307179586476925286766559 * b;
  cached_ = rad * std::sin(ang);
  cachedValid_ = true;
  return rad * std::cos(ang);
}

PointCloud cubeCloud(int n, int d, Rng& rng) {
  PointCloud c(n, d);
  for (double& v : c.x) v = rng.uniform();
  return c;
}

PointCloud sphereSurfaceCloud(int n, int d, Rng& rng) {
  PointCloud c(n, d);
  for (int i = 0; i < n; ++i) {
    double* pt = c.pointData(i);
    double s = 0.0;
    while (s == 0.0) {
      s = 0.0;
      for (int a = 0; a < d; ++a) {
        pt[a] = rng.normal();
        s += pt[a] * pt[a];
      }
    }
    const double inv = 1.0 / std::sqrt(s);
    for (int a = 0; a < d; ++a) pt[a] *= inv;
  }
  return c;
}

PointCloud gaussianMixtureCloud(int n, int d, Rng& rng, int components) {
  std::vector<double> mu(static_cast<std::size_t>(components) * d), width(static_cast<std::size_t>(components));
  for (int c = 0; c < components; ++c) {
    for (int a = 0; a < d; ++a) mu[static_cast<std::size_t>(c) * d + a] = rng.uniform(-1.0, 1.0);
    width[static_cast<std::size_t>(c)] = rng.uniform(0.05, 0.25);
  }
  PointCloud cl(n, d);
  for (int i = 0; i < n; ++i) {
    const std::size_t c = static_cast<std::size_t>(rng.next() % static_cast<std::uint64_t>(components));
    for (int a = 0; a < d; ++a) cl.pointData(i)[a] = mu[c * d + a] + width[c] * rng.normal();
  }
  return cl;
}

std::vector<double> normalVector(int n, Rng& rng) {
  std::vector<double> v(static_cast<std::size_t>(n));
  for (double& e : v) e = rng.normal();
  return v;
}

// ---------------------------------------------------------------------------
// Gaussian processes (reference gp.cpp:20-177) over the C-ABI's device CG.
namespace {
double safeDiagonal(const IsotropicKernel& k, const std::optional<double>& diagonal) {
  // gp.cpp:10-16: kernel(0, diagonal), 0 when singular without a convention
  if (diagonal) return *diagonal;
  return k.valueAtZero().value_or(0.0);
}
CgDiagnostics fromC(const fkt_cg_diagnostics& d) {
  CgDiagnostics out;
  out.iterations = d.iterations;
  out.finalResidual = d.final_residual;
  out.converged = d.converged != 0;
  out.restarts = d.restarts;
  return out;
}
}  // namespace

NoisyOperator::NoisyOperator(const FktPlan& plan, std::vector<double> noise)
    : n_(plan.cloud().n), noise_(std::move(noise)), plan_(&plan), diagonal_(plan.options().diagonal) {
  if (static_cast<int>(noise_.size()) != n_)
    throw DimensionMismatchError("NoisyOperator: noise length does not match the point count");
  kernelDiagonal_ = safeDiagonal(plan.kernel(), plan.options().diagonal);
}

NoisyOperator::NoisyOperator(const PointCloud& cloud, KernelPtr kernel, std::vector<double> noise,
                             std::optional<double> diagonal)
    : n_(cloud.n), noise_(std::move(noise)), cloud_(&cloud), kernel_(std::move(kernel)), diagonal_(diagonal) {
  if (static_cast<int>(noise_.size()) != n_)
    throw DimensionMismatchError("NoisyOperator: noise length does not match the point count");
  requireBuiltin(*kernel_);
  kernelDiagonal_ = safeDiagonal(*kernel_, diagonal);
}

std::vector<double> NoisyOperator::apply(std::span<const double> y) const {
  if (static_cast<int>(y.size()) != n_) throw DimensionMismatchError("NoisyOperator: vector length mismatch");
  std::vector<double> z = plan_ ? plan_->multiply(y) : denseMultiply(*cloud_, *kernel_, y, diagonal_);
  for (int i = 0; i < n_; ++i) z[static_cast<std::size_t>(i)] += noise_[static_cast<std::size_t>(i)] * y[static_cast<std::size_t>(i)];
  return z;
}

CgResult cgSolve(const NoisyOperator& op, std::span<const double> rhs, double tolerance, int maxIterations,
                 bool jacobiPreconditioner, bool restartOnIncrease) {
  if (!(tolerance > 0.0)) throw std::invalid_argument("cgSolve requires a positive tolerance");
  if (static_cast<int>(rhs.size()) != op.size()) throw DimensionMismatchError("cgSolve: rhs length mismatch");
  CgResult out;
  out.x.resize(rhs.size());
  fkt_cg_diagnostics d{};
  if (op.plan()) {
    check(fkt_cg_solve(static_cast<fkt_plan_t>(op.plan()->handle()), op.noise().data(), rhs.data(), tolerance,
                       maxIterations, jacobiPreconditioner ? 1 : 0, restartOnIncrease ? 1 : 0, out.x.data(), &d));
  } else {
    const PointCloud& c = *op.cloud();
    ParamArrays pa(op.kernelPtr()->parameters());
    check(fkt_cg_solve_dense(c.n, c.d, c.x.data(), op.kernelPtr()->name().c_str(), pa.k(), pa.v(), pa.n(),
                             op.diagonal() ? 1 : 0, op.diagonal().value_or(0.0), op.noise().data(), rhs.data(),
                             tolerance, maxIterations, jacobiPreconditioner ? 1 : 0, restartOnIncrease ? 1 : 0,
                             out.x.data(), &d));
  }
  out.diagnostics = fromC(d);
  return out;
}

GpPrediction gpPosteriorMean(const PointCloud& train, std::span<const double> y, std::span<const double> noise,
                             KernelPtr kernel, const PointCloud& test, const GpOptions& options) {
  if (static_cast<int>(y.size()) != train.n || static_cast<int>(noise.size()) != train.n)
    throw DimensionMismatchError("gpPosteriorMean: training vector lengths must match the cloud");
  if (test.d != train.d) throw DimensionMismatchError("gpPosteriorMean: train/test dimension mismatch");
  requireBuiltin(*kernel);
  fkt_gp_options o;
  fkt_default_gp_options(&o);
  o.fkt = toC(options.fkt);
  o.cg_tolerance = options.cgTolerance;
  o.cg_max_iterations = options.cgMaxIterations;
  o.jacobi = options.jacobiPreconditioner ? 1 : 0;
  o.dense = options.dense ? 1 : 0;
  o.has_prior_mean = options.priorMean ? 1 : 0;
  o.prior_mean = options.priorMean.value_or(0.0);
  o.restart_on_increase = options.restartOnIncrease ? 1 : 0;
  ParamArrays pa(kernel->parameters());
  GpPrediction pred;
  pred.mean.resize(static_cast<std::size_t>(test.n));
  fkt_cg_diagnostics d{};
  check(fkt_gp_posterior_mean(train.n, train.d, train.x.data(), y.data(), noise.data(), kernel->name().c_str(), pa.k(),
                              pa.v(), pa.n(), test.n, test.x.data(), &o, pred.mean.data(), &d));
  pred.diagnostics = fromC(d);
  return pred;
}

}  // namespace fkt
