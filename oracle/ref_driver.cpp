// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI + CLI driver around the UNMODIFIED reference library (the sources in
// /root/reference/proj/src compiled by oracle/Makefile into oracle/_ref/).
// Used by tests/ (parity), tests/golden/make_golden.py (fixtures) and
// bench.py --impl reference / cpu_baseline (the reference CPU arm).
//
// Exposes: the BASELINE config input recipes (built on the
// reference's own fkt::Rng, proj/include/fkt/synthetic.hpp:17-50), plan
// construction (proj/src/transform.cpp:39-92), tree/set dumps
// (proj/include/fkt/tree.hpp:30-79), multiply (transform.cpp:184-204), the
// dense oracle (transform.cpp:210-237) and sampled dense rows.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "fkt/gp.hpp"
#include "fkt/harmonics.hpp"
#include "fkt/synthetic.hpp"
#include "fkt/transform.hpp"

namespace {

thread_local std::string g_err;

fkt::IsotropicKernel::Params parseParams(const char* kv) {
  fkt::IsotropicKernel::Params params;
  if (!kv || !*kv) return params;
  std::stringstream ss(kv);
  std::string item;
  while (std::getline(ss, item, ',')) {
    const auto eq = item.find('=');
    if (eq == std::string::npos) continue;
    params[item.substr(0, eq)] = std::stod(item.substr(eq + 1));
  }
  return params;
}

struct RefPlan {
  std::unique_ptr<fkt::FktPlan> plan;
  double planSeconds = 0.0;
};

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

const char* fktref_last_error() { return g_err.c_str(); }

int fktref_config_dims(int cfg, int* d, int* nrhs) {
  static const int dims[6] = {0, 3, 3, 5, 3, 2};
  if (cfg < 1 || cfg > 5) return -1;
  *d = dims[cfg];
  *nrhs = cfg == 5 ? 16 : 1;
  return 0;
}

// SURVEY Appendix B recipes, all from fkt::Rng(seed); x is n*d row-major,
// w is n*nrhs column-major.
int fktref_gen_config(int cfg, int n, std::uint64_t seed, double* x, double* w) {
  try {
    fkt::Rng rng(seed);
    int d = 0, nrhs = 0;
    if (fktref_config_dims(cfg, &d, &nrhs) != 0) throw std::invalid_argument("bad cfg");
    const std::size_t nd = static_cast<std::size_t>(n) * d;
    if (cfg == 1 || cfg == 2) {
      fkt::PointCloud c = fkt::cubeCloud(n, 3, rng);
      std::memcpy(x, c.x.data(), nd * sizeof(double));
      auto y = fkt::normalVector(n, rng);
      std::memcpy(w, y.data(), static_cast<std::size_t>(n) * sizeof(double));
    } else if (cfg == 3) {
      double mu[8][5];
      for (int c = 0; c < 8; ++c)
        for (int a = 0; a < 5; ++a) mu[c][a] = rng.uniform();
      for (int i = 0; i < n; ++i) {
        const int c = static_cast<int>(rng.next() % 8);
        for (int a = 0; a < 5; ++a) x[static_cast<std::size_t>(i) * 5 + a] = mu[c][a] + 0.05 * rng.normal();
      }
      const double s = std::sqrt(2.0);
      for (std::size_t i = 0; i < nd; ++i) x[i] *= s;
      auto y = fkt::normalVector(n, rng);
      std::memcpy(w, y.data(), static_cast<std::size_t>(n) * sizeof(double));
    } else if (cfg == 4) {
      fkt::PointCloud c = fkt::sphereSurfaceCloud(n, 3, rng);
      for (int i = 0; i < n; ++i) {
        const double s = 1.0 + 0.01 * rng.normal();
        for (int a = 0; a < 3; ++a) c.x[static_cast<std::size_t>(i) * 3 + a] *= s;
      }
      std::memcpy(x, c.x.data(), nd * sizeof(double));
      for (int i = 0; i < n; ++i) w[i] = rng.uniform(-1.0, 1.0);
    } else {
      double mu[10][2];
      for (int c = 0; c < 10; ++c)
        for (int a = 0; a < 2; ++a) mu[c][a] = rng.uniform(-50.0, 50.0);
      for (int i = 0; i < n; ++i) {
        const int c = static_cast<int>(rng.next() % 10);
        for (int a = 0; a < 2; ++a) x[static_cast<std::size_t>(i) * 2 + a] = mu[c][a] + 3.0 * rng.normal();
      }
      for (int r = 0; r < 16; ++r) {
        auto y = fkt::normalVector(n, rng);
        std::memcpy(w + static_cast<std::size_t>(r) * n, y.data(), static_cast<std::size_t>(n) * sizeof(double));
      }
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Generic seeded generators (proj/src/synthetic.cpp).
int fktref_gen_cloud(const char* kind, int n, int d, std::uint64_t seed, double* x, double* y) {
  try {
    fkt::Rng rng(seed);
    fkt::PointCloud c;
    if (std::strcmp(kind, "cube") == 0)
      c = fkt::cubeCloud(n, d, rng);
    else if (std::strcmp(kind, "sphere") == 0)
      c = fkt::sphereSurfaceCloud(n, d, rng);
    else if (std::strcmp(kind, "mixture") == 0)
      c = fkt::gaussianMixtureCloud(n, d, rng);
    else
      throw std::invalid_argument("unknown cloud kind");
    std::memcpy(x, c.x.data(), c.x.size() * sizeof(double));
    if (y) {
      auto v = fkt::normalVector(n, rng);
      std::memcpy(y, v.data(), v.size() * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void* fktref_plan_create(int n, int d, const double* x, const char* kernel, const char* params, int p,
                         double theta, int leaf, int compression, int eager, int threads, int hasDiag,
                         double diag) {
  try {
    fkt::PointCloud cloud(n, d);
    std::memcpy(cloud.x.data(), x, static_cast<std::size_t>(n) * d * sizeof(double));
    fkt::FktOptions o;
    o.p = p;
    o.theta = theta;
    o.leafCapacity = leaf;
    // compression -1: a Barnes-Hut plan (FktOptions::barnesHut, transform.cpp:44-60)
    o.barnesHut = compression == -1;
    o.compression = compression == 1 ? fkt::CompressionMode::On
                    : compression == 2 ? fkt::CompressionMode::Off
                                       : fkt::CompressionMode::Auto;
    o.eagerOperators = eager != 0;
    o.threads = threads;
    if (hasDiag) o.diagonal = diag;
    auto k = fkt::makeKernel(kernel, parseParams(params));
    auto* rp = new RefPlan();
    const double t0 = now();
    rp->plan = std::make_unique<fkt::FktPlan>(std::move(cloud), k, o);
    rp->planSeconds = now() - t0;
    return rp;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void fktref_plan_destroy(void* h) { delete static_cast<RefPlan*>(h); }

double fktref_plan_seconds(void* h) { return static_cast<RefPlan*>(h)->planSeconds; }

int fktref_plan_info(void* h, long long* nodes, long long* farTotal, long long* nearTotal, int* compressed,
                     long long* coefCount) {
  const auto& plan = *static_cast<RefPlan*>(h)->plan;
  const auto& t = plan.tree();
  long long f = 0, nn = 0;
  for (std::size_t b = 0; b < t.nodeCount(); ++b) {
    f += static_cast<long long>(t.node(b).farSet.size());
    nn += static_cast<long long>(t.node(b).nearSet.size());
  }
  *nodes = static_cast<long long>(t.nodeCount());
  *farTotal = f;
  *nearTotal = nn;
  *compressed = plan.compressed() ? 1 : 0;
  *coefCount = static_cast<long long>(plan.coefficientCount());
  return 0;
}

// Arrays sized by fktref_plan_info; any pointer may be null to skip it.
int fktref_plan_tree(void* h, std::uint32_t* order, std::uint32_t* begin, std::uint32_t* end, int* left,
                     int* right, double* radius, double* center, double* boxLo, double* boxHi,
                     long long* farOff, std::uint32_t* far, long long* nearOff, std::uint32_t* nearList,
                     double* perm) {
  const auto& t = static_cast<RefPlan*>(h)->plan->tree();
  const int d = t.dimension();
  if (order) std::memcpy(order, t.order().data(), t.order().size() * sizeof(std::uint32_t));
  if (perm)
    for (int pos = 0; pos < t.pointCount(); ++pos) {
      auto pt = t.pointAt(static_cast<std::uint32_t>(pos));
      for (int a = 0; a < d; ++a) perm[static_cast<std::size_t>(pos) * d + a] = pt[static_cast<std::size_t>(a)];
    }
  long long fo = 0, no = 0;
  for (std::size_t b = 0; b < t.nodeCount(); ++b) {
    const auto& nd = t.node(b);
    if (begin) begin[b] = nd.begin;
    if (end) end[b] = nd.end;
    if (left) left[b] = nd.left;
    if (right) right[b] = nd.right;
    if (radius) radius[b] = nd.radius;
    for (int a = 0; a < d; ++a) {
      if (center) center[b * d + a] = nd.center[static_cast<std::size_t>(a)];
      if (boxLo) boxLo[b * d + a] = nd.boxLo[static_cast<std::size_t>(a)];
      if (boxHi) boxHi[b * d + a] = nd.boxHi[static_cast<std::size_t>(a)];
    }
    if (farOff) farOff[b] = fo;
    if (nearOff) nearOff[b] = no;
    if (far) std::memcpy(far + fo, nd.farSet.data(), nd.farSet.size() * sizeof(std::uint32_t));
    if (nearList) std::memcpy(nearList + no, nd.nearSet.data(), nd.nearSet.size() * sizeof(std::uint32_t));
    fo += static_cast<long long>(nd.farSet.size());
    no += static_cast<long long>(nd.nearSet.size());
  }
  if (farOff) farOff[t.nodeCount()] = fo;
  if (nearOff) nearOff[t.nodeCount()] = no;
  return 0;
}

// z = K y for nrhs column-major right-hand sides (one reference multiply per
// column: the reference API is single-RHS, transform.hpp:47).
int fktref_plan_multiply(void* h, const double* y, double* z, int nrhs) {
  try {
    const auto& plan = *static_cast<RefPlan*>(h)->plan;
    const std::size_t n = static_cast<std::size_t>(plan.cloud().n);
    for (int r = 0; r < nrhs; ++r) {
      auto out = plan.multiply(std::span<const double>(y + r * n, n));
      std::memcpy(z + r * n, out.data(), n * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int fktref_dense(int n, int d, const double* x, const char* kernel, const char* params, const double* y,
                 double* z, int threads, int hasDiag, double diag) {
  try {
    fkt::PointCloud cloud(n, d);
    std::memcpy(cloud.x.data(), x, static_cast<std::size_t>(n) * d * sizeof(double));
    auto k = fkt::makeKernel(kernel, parseParams(params));
    std::optional<double> dg;
    if (hasDiag) dg = diag;
    auto out = fkt::denseMultiply(cloud, *k, std::span<const double>(y, static_cast<std::size_t>(n)), dg, threads);
    std::memcpy(z, out.data(), out.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// --- reference GP / CG (gp.cpp) ---------------------------------------------
namespace {
// test_gp.cpp:14-18: the zero kernel (a user lambda the GPU path cannot run)
fkt::KernelPtr refKernel(const char* name, const char* params) {
  if (std::string(name) == "zero")
    return std::make_shared<fkt::IsotropicKernel>(
        "zero", fkt::IsotropicKernel::Params{}, [](double) { return 0.0; },
        [](const fkt::Jet& r) { return fkt::Jet::constant(0.0, r.center(), r.order()); }, std::nullopt, 0.0);
  return fkt::makeKernel(name, parseParams(params));
}
void putDiag(const fkt::CgDiagnostics& dg, int* it, double* res, int* conv, int* rs) {
  *it = dg.iterations;
  *res = dg.finalResidual;
  *conv = dg.converged ? 1 : 0;
  *rs = dg.restarts;
}
}  // namespace

// cgSolve (gp.cpp:58-124) over NoisyOperator(plan, noise) when usePlan, else
// the dense NoisyOperator(cloud, kernel, noise, diagonal).
int fktref_cg_solve(int n, int d, const double* x, const char* kernel, const char* params, int usePlan, int p,
                    double theta, int leaf, int hasDiag, double diag, const double* noise, const double* rhs,
                    double tol, int maxit, int jacobi, double* out, int* it, double* res, int* conv, int* rs) {
  try {
    fkt::PointCloud cloud(n, d);
    std::memcpy(cloud.x.data(), x, static_cast<std::size_t>(n) * d * sizeof(double));
    auto k = refKernel(kernel, params);
    std::optional<double> dg;
    if (hasDiag) dg = diag;
    std::vector<double> nz(noise, noise + n);
    std::unique_ptr<fkt::FktPlan> plan;
    std::unique_ptr<fkt::NoisyOperator> op;
    if (usePlan) {
      fkt::FktOptions o;
      o.p = p;
      o.theta = theta;
      o.leafCapacity = leaf;
      o.diagonal = dg;
      plan = std::make_unique<fkt::FktPlan>(cloud, k, o);
      op = std::make_unique<fkt::NoisyOperator>(*plan, nz);
    } else {
      op = std::make_unique<fkt::NoisyOperator>(cloud, k, nz, dg);
    }
    const auto r = fkt::cgSolve(*op, std::span<const double>(rhs, static_cast<std::size_t>(n)), tol, maxit, jacobi != 0);
    std::memcpy(out, r.x.data(), r.x.size() * sizeof(double));
    putDiag(r.diagnostics, it, res, conv, rs);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// gpPosteriorMean (gp.cpp:126-177).
int fktref_gp_posterior_mean(int nTrain, int d, const double* trainX, const double* y, const double* noise,
                             const char* kernel, const char* params, int nTest, const double* testX, int p,
                             double theta, int leaf, int hasDiag, double diag, double tol, int maxit, int jacobi,
                             int dense, int hasPrior, double prior, double* mean, int* it, double* res, int* conv,
                             int* rs) {
  try {
    fkt::PointCloud train(nTrain, d), test(nTest, d);
    std::memcpy(train.x.data(), trainX, static_cast<std::size_t>(nTrain) * d * sizeof(double));
    if (nTest > 0) std::memcpy(test.x.data(), testX, static_cast<std::size_t>(nTest) * d * sizeof(double));
    fkt::GpOptions o;
    o.fkt.p = p;
    o.fkt.theta = theta;
    o.fkt.leafCapacity = leaf;
    if (hasDiag) o.fkt.diagonal = diag;
    o.cgTolerance = tol;
    o.cgMaxIterations = maxit;
    o.jacobiPreconditioner = jacobi != 0;
    o.dense = dense != 0;
    if (hasPrior) o.priorMean = prior;
    const auto pr = fkt::gpPosteriorMean(train, std::span<const double>(y, static_cast<std::size_t>(nTrain)),
                                         std::span<const double>(noise, static_cast<std::size_t>(nTrain)),
                                         refKernel(kernel, params), test, o);
    std::memcpy(mean, pr.mean.data(), pr.mean.size() * sizeof(double));
    putDiag(pr.diagnostics, it, res, conv, rs);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Rows `rows[0..m)` of the dense product, with the same per-pair arithmetic
// as denseMultiply (transform.cpp:218-233), parallel over rows.
int fktref_dense_rows(int n, int d, const double* x, const char* kernel, const char* params, const double* y,
                      int m, const std::int64_t* rows, double* z, int threads, int hasDiag, double diag) {
  try {
    auto k = fkt::makeKernel(kernel, parseParams(params));
    std::optional<double> dg;
    if (hasDiag) dg = diag;
    const int T = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> pool;
    std::exception_ptr err;
    for (int w = 0; w < T; ++w)
      pool.emplace_back([&, w] {
        try {
          for (int q = w; q < m; q += T) {
            const double* pi = x + rows[q] * d;
            double acc = 0.0;
            for (int j = 0; j < n; ++j) {
              const double* pj = x + static_cast<std::size_t>(j) * d;
              double dist2 = 0.0;
              for (int a = 0; a < d; ++a) {
                const double t = pi[a] - pj[a];
                dist2 += t * t;
              }
              const double r = std::sqrt(dist2);
              acc += (*k)(r, r == 0.0 ? dg : std::nullopt) * y[j];
            }
            z[q] = acc;
          }
        } catch (...) {
          err = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Exact T-bar_kjm of the reference table (coefficients.cpp:102-106) as
// "num/den", and its double (tbarDouble, :108-111).
int fktref_tbar(int d, int p, int k, int j, int m, double* value, char* buf, int len) {
  try {
    const auto& t = fkt::coefficientTable(d, p);
    const auto& q = t.tbar(k, j, m);
    *value = t.tbarDouble(k, j, m);
    std::ostringstream os;
    os << numerator(q) << "/" << denominator(q);
    std::snprintf(buf, static_cast<std::size_t>(len), "%s", os.str().c_str());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CoefficientTable::serialize (coefficients.cpp:113-124); returns the length
// needed including the NUL.
long long fktref_tbar_serialize(int d, int p, char* buf, long long len) {
  try {
    const std::string s = fkt::coefficientTable(d, p).serialize();
    if (buf && len > 0) std::snprintf(buf, static_cast<std::size_t>(len), "%s", s.c_str());
    return static_cast<long long>(s.size()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CoefficientTable::deserialize (:126-166): 1 parses and equals the computed
// table, 0 parses but differs, -1 nullopt.
int fktref_tbar_deserialize(const char* text) {
  auto t = fkt::CoefficientTable::deserialize(text);
  if (!t) return -1;
  if (t->maxOrder() > fkt::kMaxExpansionOrder) return 0;
  return *t == fkt::coefficientTable(t->dimension(), t->maxOrder()) ? 1 : 0;
}

// Compression ranks per degree (expansion.cpp:190-243).
int fktref_compression_ranks(const char* kernel, const char* params, int d, int p, int* ranks) {
  try {
    auto k = fkt::makeKernel(kernel, parseParams(params));
    auto f = fkt::radialCompression(*k, fkt::coefficientTable(d, p), p);
    for (int i = 0; i <= p; ++i) ranks[i] = f[static_cast<std::size_t>(i)].rank;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Z_k (harmonics.cpp:114-116) and the orthonormal harmonic values at a point
// (harmonics.cpp:160-246), degree-major.
double fktref_addition_normalizer(int d, int k) { return fkt::additionNormalizer(d, k); }

int fktref_harmonics(int d, int p, const double* point, double* values) {
  try {
    fkt::HarmonicBasis basis(d, p);
    std::vector<double> v;
    basis.evaluate(std::span<const double>(point, static_cast<std::size_t>(d)), v);
    std::memcpy(values, v.data(), v.size() * sizeof(double));
    return static_cast<int>(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Kernel value and jet (kernels.hpp:49-64) for the builtin kernels.
int fktref_kernel_jet(const char* kernel, const char* params, double r, int order, double* c) {
  try {
    auto k = fkt::makeKernel(kernel, parseParams(params));
    const fkt::Jet j = k->jetAt(r, order);
    for (int m = 0; m <= order; ++m) c[m] = j.coeff(m);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// SURVEY Appendix A fingerprints (64-bit FNV-1a folds).
int fktref_fingerprints(void* h, std::uint64_t* orderHash, std::uint64_t* setsHash, std::uint64_t* geomHash) {
  const auto& t = static_cast<RefPlan*>(h)->plan->tree();
  const std::uint64_t P = 1099511628211ull;
  std::uint64_t ho = 1469598103934665603ull, hs = ho, hg = ho;
  for (std::uint32_t v : t.order()) {
    ho ^= v;
    ho *= P;
  }
  for (std::size_t b = 0; b < t.nodeCount(); ++b) {
    const auto& nd = t.node(b);
    for (std::uint32_t v : nd.farSet) {
      hs ^= v + b * 0x9e3779b97f4a7c15ull;
      hs *= P;
    }
    for (std::uint32_t v : nd.nearSet) {
      hs ^= static_cast<std::uint64_t>(v) * 31 + b;
      hs *= P;
    }
    std::uint64_t bits;
    std::memcpy(&bits, &nd.radius, 8);
    hg ^= bits;
    hg *= P;
    for (double c : nd.center) {
      std::memcpy(&bits, &c, 8);
      hg ^= bits;
      hg *= P;
    }
  }
  *orderHash = ho;
  *setsHash = hs;
  *geomHash = hg;
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// CLI: fkt_ref --cfg K [--n N] [--threads T] [--reps R] [--eager 0|1]
// Prints one JSON line: fingerprints, plan seconds, median MVM seconds.
#ifdef FKTREF_MAIN
int main(int argc, char** argv) {
  int cfg = 1, n = -1, threads = 0, reps = 1, eager = -1;
  for (int i = 1; i + 1 < argc; i += 2) {
    std::string a = argv[i];
    if (a == "--cfg") cfg = std::atoi(argv[i + 1]);
    else if (a == "--n") n = std::atoi(argv[i + 1]);
    else if (a == "--threads") threads = std::atoi(argv[i + 1]);
    else if (a == "--reps") reps = std::atoi(argv[i + 1]);
    else if (a == "--eager") eager = std::atoi(argv[i + 1]);
  }
  static const int Ns[6] = {0, 20000, 1000000, 1000000, 4000000, 2000000};
  static const char* K[6] = {"", "cauchy", "matern32", "gaussian", "inverse-r", "cauchy"};
  static const char* Pm[6] = {"", "sigma=1", "sigma=1,rho=0.1", "", "", "sigma=1"};
  static const int ps[6] = {0, 4, 6, 4, 8, 6};
  static const int leafs[6] = {0, 512, 512, 1024, 512, 512};
  static const double thetas[6] = {0, 0.5, 0.5, 0.75, 0.5, 0.75};
  if (n < 0) n = Ns[cfg];
  int d, nrhs;
  fktref_config_dims(cfg, &d, &nrhs);
  std::vector<double> x(static_cast<std::size_t>(n) * d), w(static_cast<std::size_t>(n) * nrhs);
  fktref_gen_config(cfg, n, 42, x.data(), w.data());
  if (eager < 0) eager = n < 100000;
  void* h = fktref_plan_create(n, d, x.data(), K[cfg], Pm[cfg], ps[cfg], thetas[cfg], leafs[cfg], 0, eager,
                               threads, 0, 0.0);
  if (!h) {
    std::fprintf(stderr, "plan failed: %s\n", fktref_last_error());
    return 1;
  }
  std::uint64_t ho, hs, hg;
  fktref_fingerprints(h, &ho, &hs, &hg);
  long long nodes, ft, nt, cc;
  int comp;
  fktref_plan_info(h, &nodes, &ft, &nt, &comp, &cc);
  std::vector<double> z(w.size());
  std::vector<double> times;
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    fktref_plan_multiply(h, w.data(), z.data(), nrhs);
    times.push_back(now() - t0);
  }
  std::sort(times.begin(), times.end());
  if (times.empty()) times.push_back(0.0);
  double zs = 0;
  for (double v : z) zs += v;
  std::printf(
      "{\"cfg\": %d, \"n\": %d, \"nodes\": %lld, \"far_total\": %lld, \"near_total\": %lld, \"compressed\": %d, "
      "\"coef\": %lld, \"order\": \"%016llx\", \"sets\": \"%016llx\", \"geom\": \"%016llx\", \"plan_s\": %.4f, "
      "\"mvm_s\": %.4f, \"zsum\": %.17g}\n",
      cfg, n, nodes, ft, nt, comp, cc, (unsigned long long)ho, (unsigned long long)hs, (unsigned long long)hg,
      fktref_plan_seconds(h), times[times.size() / 2], zs);
  fktref_plan_destroy(h);
  return 0;
}
#endif
