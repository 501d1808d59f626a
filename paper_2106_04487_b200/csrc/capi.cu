// C-ABI implementation (include/fkt_cuda.h). Converts exceptions into status
// codes + a thread-local message; every entry point is a thin shell over the
// plan / tree / kernel code in this directory.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>

#include "../../include/fkt_cuda.h"
#include "gp.hpp"
#include "plan.hpp"

namespace fktb {
void synthCloud(const std::string& kind, int n, int d, std::uint64_t seed, double* x, double* y);
void synthConfig(int cfg, int n, std::uint64_t seed, double* x, double* w);
int configDims(int cfg, int* d, int* nrhs);
}  // namespace fktb

struct fkt_tree_s {
  fktb::DeviceTree* tree = nullptr;   // borrowed or owned
  std::unique_ptr<fktb::DeviceTree> owned;
  cudaStream_t ownedStream = nullptr;
  // lazily materialised reference-form sets
  bool farReady = false, nearReady = false;
  std::vector<long long> farOff, nearOff;
  std::vector<uint32_t> farIdx, nearIdx;
  std::mutex mutex;
};
struct fkt_plan_s {
  std::unique_ptr<fktb::DevicePlan> plan;
  bool cached = false;  // owned by the plan cache (fkt_plan_cache_get)
  int refs = 0;         // outstanding fkt_plan_cache_get references
  // borrowed tree view (fkt_plan_tree): lives and dies with this handle, so a
  // freed plan never leaves a view (and its materialised sets) behind
  std::unique_ptr<fkt_tree_s> view;
  std::mutex viewMutex;
};

namespace {

thread_local std::string g_msg;
thread_local int g_code = FKT_OK;

struct DimensionMismatch : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct Unsupported : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct OrderTooLarge : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ZeroReference : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

int fail(int code, const char* msg) {
  g_code = code;
  g_msg = msg;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    g_code = FKT_OK;
    g_msg.clear();
    f();
    return FKT_OK;
  } catch (const DimensionMismatch& e) {
    return fail(FKT_ERR_DIMENSION_MISMATCH, e.what());
  } catch (const Unsupported& e) {
    return fail(FKT_ERR_UNSUPPORTED, e.what());
  } catch (const OrderTooLarge& e) {
    return fail(FKT_ERR_ORDER_TOO_LARGE, e.what());
  } catch (const ZeroReference& e) {
    return fail(FKT_ERR_ZERO_REFERENCE, e.what());
  } catch (const fktb::NotRecurrenceKernelError& e) {
    return fail(FKT_ERR_NOT_RECURRENCE, e.what());
  } catch (const fktb::CudaError& e) {
    return fail(FKT_ERR_CUDA, e.what());
  } catch (const std::invalid_argument& e) {
    const std::string m = e.what();
    if (m.find("unsupported on the GPU path") != std::string::npos) return fail(FKT_ERR_UNSUPPORTED, e.what());
    if (m.find("exceeds the supported cap") != std::string::npos) return fail(FKT_ERR_ORDER_TOO_LARGE, e.what());
    return fail(FKT_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::domain_error& e) {
    return fail(FKT_ERR_SINGULAR_AT_ZERO, e.what());
  } catch (const std::exception& e) {
    return fail(FKT_ERR_INTERNAL, e.what());
  } catch (...) {
    return fail(FKT_ERR_INTERNAL, "unknown error");
  }
}

std::map<std::string, double> toParams(const char* const* keys, const double* values, int np) {
  std::map<std::string, double> p;
  for (int i = 0; i < np; ++i) p[keys[i]] = values[i];
  return p;
}

fktb::KernelSpec spec(const char* name, const char* const* keys, const double* values, int np) {
  if (!name) throw std::invalid_argument("kernel name is null");
  return fktb::makeKernelSpec(name, toParams(keys, values, np));
}

void requireDevice() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw fktb::CudaError("no CUDA device available: the FKT MVM has no CPU fallback");
}

}  // namespace

extern "C" {

const char* fkt_last_error(void) { return g_msg.c_str(); }
int fkt_last_error_code(void) { return g_code; }
const char* fkt_version(void) { return "fkt-b200 0.1 (sm_100a)"; }
int fkt_kernel_count(void) { return FKTB_KERNEL_COUNT; }
const char* fkt_kernel_name(int i) {
  static const std::vector<std::string> names = fktb::builtinKernelNames();
  return i >= 0 && i < static_cast<int>(names.size()) ? names[static_cast<size_t>(i)].c_str() : nullptr;
}

int fkt_kernel_check(const char* name, const char* const* keys, const double* values, int nparams,
                     int* has_recurrence, int* has_value_at_zero, double* value_at_zero) {
  return guarded([&] {
    auto k = spec(name, keys, values, nparams);
    if (has_recurrence) *has_recurrence = k.recurrence ? 1 : 0;
    if (has_value_at_zero) *has_value_at_zero = k.valueAtZero ? 1 : 0;
    if (value_at_zero) *value_at_zero = k.valueAtZero.value_or(0.0);
  });
}

int fkt_kernel_eval(const char* name, const char* const* keys, const double* values, int nparams, const double* r,
                    double* out, long long count, int has_diagonal, double diagonal) {
  return guarded([&] {
    auto k = spec(name, keys, values, nparams);
    for (long long i = 0; i < count; ++i) {
      if (r[i] == 0.0) {
        if (has_diagonal)
          out[i] = diagonal;
        else if (k.valueAtZero)
          out[i] = *k.valueAtZero;
        else
          throw std::domain_error("kernel '" + k.name + "' is singular at r = 0 and no diagonal convention is set");
      } else {
        out[i] = fktb::kernelEvalHost(k, r[i]);
      }
    }
  });
}

int fkt_kernel_recurrence(const char* name, const char* const* keys, const double* values, int nparams, int* terms,
                          int* powers, int max_terms, char* buf, long long buf_len) {
  return guarded([&] {
    const fktb::KernelSpec k = fktb::makeKernelSpec(name, toParams(keys, values, nparams));
    *terms = 0;
    if (!k.recurrence) return;
    std::string text;
    int i = 0;
    for (const auto& [p, c] : k.recurrence->terms()) {
      if (i >= max_terms) throw std::invalid_argument("recurrence: more terms than max_terms");
      powers[i++] = p;
      text += c.num().str() + "/" + c.den().str();
      text.push_back('\0');
    }
    if (static_cast<long long>(text.size()) > buf_len) throw std::invalid_argument("recurrence: buffer too small");
    std::memcpy(buf, text.data(), text.size());
    *terms = i;
  });
}

int fkt_kernel_eval_jet(const char* name, const char* const* keys, const double* values, int nparams, double center,
                        int order, const double* in, double* out) {
  return guarded([&] {
    const fktb::KernelSpec k = fktb::makeKernelSpec(name, toParams(keys, values, nparams));
    fkt::Jet arg(center, order);
    for (int i = 0; i <= order; ++i) arg.coeff(i) = in[i];
    const fkt::Jet r = fktb::kernelJetHost(k, arg);
    for (int i = 0; i <= order; ++i) out[i] = r.coeff(i);
  });
}

void fkt_default_options(fkt_options* o) {
  o->p = 4;
  o->theta = 0.75;
  o->leaf_capacity = 512;
  o->compression = FKT_COMPRESSION_AUTO;
  o->eager_operators = 1;
  o->barnes_hut = 0;
  o->threads = 0;
  o->has_diagonal = 0;
  o->diagonal = 0.0;
  o->near_precision = 64;
  o->deterministic = 0;
}

}  // extern "C"

namespace {
fktb::PlanOptions toPlanOptions(const fkt_options* opt) {
  fkt_options def;
  fkt_default_options(&def);
  const fkt_options& o = opt ? *opt : def;
  fktb::PlanOptions po;
  po.p = o.p;
  po.theta = o.theta;
  po.leafCapacity = o.leaf_capacity;
  po.compression = o.compression;
  po.eagerOperators = o.eager_operators != 0;
  po.barnesHut = o.barnes_hut != 0;
  po.threads = o.threads;
  po.hasDiagonal = o.has_diagonal != 0;
  po.diagonal = o.diagonal;
  if (o.near_precision != 64 && o.near_precision != 32)
    throw std::invalid_argument("near_precision must be 64 or 32");
  po.nearPrecision = o.near_precision;
  po.deterministic = o.deterministic != 0;
  if (!po.barnesHut && po.p > fktb::kMaxExpansionOrder)
    throw OrderTooLarge("expansion order " + std::to_string(po.p) + " exceeds the supported cap " +
                        std::to_string(fktb::kMaxExpansionOrder));
  return po;
}

void toC(const fktb::CgDiagnostics& d, fkt_cg_diagnostics* out) {
  if (!out) return;
  out->iterations = d.iterations;
  out->final_residual = d.finalResidual;
  out->converged = d.converged ? 1 : 0;
  out->restarts = d.restarts;
}
}  // namespace

extern "C" {

int fkt_plan_create(int n, int d, const double* x, const char* kernel, const char* const* keys, const double* values,
                    int nparams, const fkt_options* opt, fkt_plan_t* out) {
  *out = nullptr;
  return guarded([&] {
    auto k = spec(kernel, keys, values, nparams);
    const fktb::PlanOptions po = toPlanOptions(opt);
    requireDevice();
    auto h = std::make_unique<fkt_plan_s>();
    h->plan = fktb::createPlan(n, d, x, k, po);
    *out = h.release();
  });
}

int fkt_plan_destroy(fkt_plan_t plan) {
  return guarded([&] {
    if (!plan) return;
    if (plan->cached) throw std::invalid_argument("plan is owned by the plan cache: use fkt_plan_cache_release");
    fktb::DevicePlan* p = plan->plan.release();
    fktb::destroyPlan(p);
    delete plan;
  });
}

}  // extern "C"

namespace {
void rebuildGuarded(fkt_plan_t plan, const double* x, bool onDevice) {
  if (!plan || !x) throw std::invalid_argument("rebuild: null plan or coordinates");
  if (plan->cached) throw std::invalid_argument("plan is shared by the plan cache: rebuild a plan of your own");
  auto& p = *plan->plan;
  std::lock_guard<std::mutex> lock(p.mutex);
  fktb::rebuildPlan(p, x, onDevice);
  std::lock_guard<std::mutex> vlock(plan->viewMutex);
  if (plan->view) {  // the borrowed tree view's materialised sets are stale
    std::lock_guard<std::mutex> tl(plan->view->mutex);
    plan->view->farReady = plan->view->nearReady = false;
  }
}
}  // namespace

extern "C" {

int fkt_plan_rebuild(fkt_plan_t plan, const double* x) {
  return guarded([&] { rebuildGuarded(plan, x, false); });
}

int fkt_plan_rebuild_device(fkt_plan_t plan, const double* x_dev) {
  return guarded([&] { rebuildGuarded(plan, x_dev, true); });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Plan cache: identical (cloud, kernel, options) requests share
// one device plan. Entries are matched on the full inputs (the coordinates
// are compared bytewise, not only hashed); unreferenced plans are kept up to
// the capacity and evicted least-recently-used first.
namespace {
struct CacheEntry {
  int n = 0, d = 0;
  std::vector<double> x;
  std::string kernel;
  std::map<std::string, double> params;
  fkt_options opt{};
  fkt_plan_t plan = nullptr;
  unsigned long long lastUse = 0;
};
std::mutex g_cacheMutex;
std::vector<CacheEntry> g_cache;
int g_cacheCapacity = 4;
unsigned long long g_cacheClock = 0;

bool sameOptions(const fkt_options& a, const fkt_options& b) {
  return a.p == b.p && a.theta == b.theta && a.leaf_capacity == b.leaf_capacity && a.compression == b.compression &&
         a.barnes_hut == b.barnes_hut && a.has_diagonal == b.has_diagonal &&
         (!a.has_diagonal || a.diagonal == b.diagonal) && a.near_precision == b.near_precision &&
         (a.deterministic != 0) == (b.deterministic != 0);
}

void evictLocked() {
  // drop unreferenced entries, oldest first, while over capacity
  while (true) {
    int unref = 0;
    for (const auto& e : g_cache) unref += e.plan->refs == 0;
    if (static_cast<int>(g_cache.size()) <= g_cacheCapacity || unref == 0) return;
    auto victim = g_cache.end();
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
      if (it->plan->refs == 0 && (victim == g_cache.end() || it->lastUse < victim->lastUse)) victim = it;
    fktb::DevicePlan* p = victim->plan->plan.release();
    fktb::destroyPlan(p);
    delete victim->plan;
    g_cache.erase(victim);
  }
}
}  // namespace

extern "C" {

int fkt_plan_cache_get(int n, int d, const double* x, const char* kernel, const char* const* keys,
                       const double* values, int nparams, const fkt_options* opt, fkt_plan_t* out, int* hit) {
  *out = nullptr;
  return guarded([&] {
    auto k = spec(kernel, keys, values, nparams);
    fkt_options o;
    fkt_default_options(&o);
    if (opt) o = *opt;
    const auto params = toParams(keys, values, nparams);
    std::lock_guard<std::mutex> lock(g_cacheMutex);
    for (auto& e : g_cache) {
      if (e.n == n && e.d == d && e.kernel == kernel && e.params == params && sameOptions(e.opt, o) &&
          std::memcmp(e.x.data(), x, static_cast<size_t>(n) * d * sizeof(double)) == 0) {
        ++e.plan->refs;
        e.lastUse = ++g_cacheClock;
        *out = e.plan;
        if (hit) *hit = 1;
        return;
      }
    }
    const fktb::PlanOptions po = toPlanOptions(&o);
    requireDevice();
    auto h = std::make_unique<fkt_plan_s>();
    h->plan = fktb::createPlan(n, d, x, k, po);
    h->cached = true;
    h->refs = 1;
    CacheEntry e;
    e.n = n;
    e.d = d;
    e.x.assign(x, x + static_cast<size_t>(n) * d);
    e.kernel = kernel;
    e.params = params;
    e.opt = o;
    e.plan = h.release();
    e.lastUse = ++g_cacheClock;
    g_cache.push_back(std::move(e));
    *out = g_cache.back().plan;
    if (hit) *hit = 0;
    evictLocked();
  });
}

int fkt_plan_cache_release(fkt_plan_t plan) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(g_cacheMutex);
    if (!plan || !plan->cached) throw std::invalid_argument("plan was not obtained from the plan cache");
    if (plan->refs <= 0) throw std::invalid_argument("plan cache reference released twice");
    --plan->refs;
    evictLocked();
  });
}

int fkt_plan_cache_set_capacity(int plans) {
  return guarded([&] {
    if (plans < 0) throw std::invalid_argument("plan cache capacity must be >= 0");
    std::lock_guard<std::mutex> lock(g_cacheMutex);
    g_cacheCapacity = plans;
    evictLocked();
  });
}

int fkt_plan_cache_size(void) {
  std::lock_guard<std::mutex> lock(g_cacheMutex);
  return static_cast<int>(g_cache.size());
}

int fkt_plan_info_get(fkt_plan_t plan, fkt_plan_info* info) {
  return guarded([&] {
    const auto& p = *plan->plan;
    const auto& t = *p.tree;
    info->n = p.n;
    info->d = p.d;
    info->p = p.options.p;
    info->nodes = t.nodes;
    long long leaves = 0;
    for (int b = 0; b < t.nodes; ++b) leaves += t.left[static_cast<size_t>(b)] < 0;
    info->leaves = leaves;
    info->depth = t.depth;
    info->far_total = t.farTotal;
    info->near_total = t.nearTotal;
    info->coefficient_count = p.far->Pref;
    info->stored_coefficients = p.P;
    info->compressed = p.compressed ? 1 : 0;
    info->plan_seconds = p.planSeconds;
    info->far_tiles = static_cast<long long>(p.farTilesHost.size());
    info->near_tiles = static_cast<long long>(p.nearTilesHost.size());
    info->s2m_tiles = static_cast<long long>(p.s2mTilesHost.size());
    info->m2t_cartesian = p.cartP > 0 ? 1 : 0;
  });
}

int fkt_plan_phases(fkt_plan_t plan, double* seconds, int count) {
  return guarded([&] {
    for (int i = 0; i < count && i < fktb::kPhaseCount; ++i) seconds[i] = plan->plan->phaseSeconds[i];
  });
}

int fkt_plan_multiply(fkt_plan_t plan, const double* y, double* z, int nrhs) {
  return guarded([&] {
    if (nrhs < 1) throw DimensionMismatch("multiply: nrhs must be >= 1");
    auto& p = *plan->plan;
    std::lock_guard<std::mutex> lock(p.mutex);
    fktb::multiplyHost(p, y, z, nrhs);
  });
}

int fkt_plan_multiply_device(fkt_plan_t plan, const double* y_dev, double* z_dev, int nrhs, void* stream) {
  return guarded([&] {
    if (nrhs < 1) throw DimensionMismatch("multiply: nrhs must be >= 1");
    auto& p = *plan->plan;
    std::lock_guard<std::mutex> lock(p.mutex);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    fktb::multiplyDevice(p, y_dev, z_dev, nrhs, st);
    if (!stream) FKTB_CUDA(cudaStreamSynchronize(st));
  });
}

int fkt_plan_stage_device(fkt_plan_t plan, int stage, const double* y_dev, double* z_dev, int nrhs, void* stream) {
  return guarded([&] {
    auto& p = *plan->plan;
    std::lock_guard<std::mutex> lock(p.mutex);
    if (nrhs < 1) throw DimensionMismatch("stage: nrhs must be >= 1");
    if (nrhs > fktb::maxRhsPerPass(p)) throw std::invalid_argument("stage: nrhs exceeds one pass; use multiply");
    if (stage == 0) fktb::ensureWorkspace(p, nrhs);
    if (nrhs > p.nrhsCap) throw std::invalid_argument("stage: run stage 0 (or a multiply) with this nrhs first");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    fktb::orderAfterPrevious(p, st);
    switch (stage) {
      case 0:
        fktb::launchGatherY(p, y_dev, p.dYp.get(), nrhs, st);
        FKTB_CUDA(cudaMemsetAsync(p.dZp.get(), 0, static_cast<size_t>(p.n) * nrhs * sizeof(double), st));
        FKTB_CUDA(cudaMemsetAsync(p.dMoments.get(), 0,
                                  static_cast<size_t>(p.tree->nodes) * fktb::momentStrideMax(p) * nrhs * sizeof(double), st));
        break;
      case 1: fktb::launchS2MAny(p, p.dYp.get(), p.dMoments.get(), nrhs, st); break;
      case 2: fktb::launchNearAny(p, p.dYp.get(), p.dZp.get(), nrhs, st); break;
      case 3:
        fktb::launchM2T(p, p.dMoments.get(), p.dZp.get(), nrhs, st);
        if (p.options.deterministic) fktb::launchDetReduce(p, nullptr, nrhs, true, st);
        break;
      case 4:
        if (p.options.deterministic) fktb::launchDetReduce(p, p.dZp.get(), nrhs, false, st);
        fktb::launchScatterZ(p, p.dZp.get(), z_dev, nrhs, st);
        break;
      default: throw std::invalid_argument("stage must be 0..4");
    }
    fktb::markDone(p, st);
    if (!stream) FKTB_CUDA(cudaStreamSynchronize(st));
  });
}

int fkt_plan_set_shard(fkt_plan_t plan, int shard, int shards) {
  return guarded([&] {
    auto& p = *plan->plan;
    std::lock_guard<std::mutex> lock(p.mutex);
    fktb::setShard(p, shard, shards);
  });
}

int fkt_plan_multiply_sharded(fkt_plan_t plan, const double* y_dev, double* z_dev, int nrhs, void* nccl_comm,
                              void* stream) {
  return guarded([&] {
    if (nrhs < 1) throw DimensionMismatch("multiply: nrhs must be >= 1");
    if (!nccl_comm) throw std::invalid_argument("sharded multiply: null communicator");
    auto& p = *plan->plan;
    std::lock_guard<std::mutex> lock(p.mutex);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : p.stream;
    fktb::multiplySharded(p, y_dev, z_dev, nrhs, nccl_comm, st);
    if (!stream) FKTB_CUDA(cudaStreamSynchronize(st));
  });
}

int fkt_nccl_unique_id(char* id128) {
  return guarded([&] { fktb::ncclUniqueIdBytes(id128); });
}

int fkt_nccl_comm_create(const char* id128, int nranks, int rank, void** comm) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("nccl comm: 0 <= rank < nranks");
    *comm = fktb::ncclCommCreate(id128, nranks, rank);
  });
}

int fkt_nccl_comm_destroy(void* comm) {
  return guarded([&] { fktb::ncclCommRelease(comm); });
}

int fkt_plan_shard_range(fkt_plan_t plan, long long* pos_lo, long long* pos_hi) {
  return guarded([&] {
    *pos_lo = plan->plan->shardLo;
    *pos_hi = plan->plan->shardHi;
  });
}

int fkt_plan_moments_device(fkt_plan_t plan, double** moments, long long* count_per_rhs) {
  return guarded([&] {
    *moments = plan->plan->dMoments.get();
    // the widest row layout (single-RHS passes may hold the Cartesian M2T
    // coefficients): stage 0 zeroes this whole range
    *count_per_rhs = static_cast<long long>(plan->plan->tree->nodes) * fktb::momentStrideMax(*plan->plan);
  });
}

void fkt_default_gp_options(fkt_gp_options* o) {
  fkt_default_options(&o->fkt);
  o->cg_tolerance = 1e-10;
  o->cg_max_iterations = 1000;
  o->jacobi = 0;
  o->dense = 0;
  o->has_prior_mean = 0;
  o->prior_mean = 0.0;
  o->restart_on_increase = 1;
}

int fkt_cg_solve(fkt_plan_t plan, const double* noise, const double* rhs, double tolerance, int max_iterations,
                 int jacobi, int restart_on_increase, double* x, fkt_cg_diagnostics* diag) {
  return guarded([&] {
    auto& p = *plan->plan;
    std::lock_guard<std::mutex> lock(p.mutex);
    if (!(tolerance > 0.0)) throw std::invalid_argument("cgSolve requires a positive tolerance");
    fktb::DeviceNoisyOperator op;
    op.n = p.n;
    op.plan = &p;
    op.kernelDiagonal = fktb::safeKernelDiagonal(p.kernel, p.options.hasDiagonal, p.options.diagonal);
    cudaStream_t st = p.stream;  // the plan's stream: its captured MVM graph is reused across solves
    const size_t bytes = static_cast<size_t>(p.n) * sizeof(double);
    op.noise.resize(static_cast<size_t>(p.n));
    fktb::DeviceBuffer<double> dRhs(static_cast<size_t>(p.n)), dX(static_cast<size_t>(p.n));
    FKTB_CUDA(cudaMemcpyAsync(op.noise.get(), noise, bytes, cudaMemcpyHostToDevice, st));
    FKTB_CUDA(cudaMemcpyAsync(dRhs.get(), rhs, bytes, cudaMemcpyHostToDevice, st));
    const auto d = fktb::cgSolveDevice(op, dRhs.get(), tolerance, max_iterations, jacobi != 0, dX.get(), st,
                                       restart_on_increase != 0);
    FKTB_CUDA(cudaMemcpyAsync(x, dX.get(), bytes, cudaMemcpyDeviceToHost, st));
    FKTB_CUDA(cudaStreamSynchronize(st));
    toC(d, diag);
  });
}

int fkt_cg_solve_dense(int n, int d, const double* points, const char* kernel, const char* const* keys,
                       const double* values, int nparams, int has_diagonal, double diagonal, const double* noise,
                       const double* rhs, double tolerance, int max_iterations, int jacobi, int restart_on_increase,
                       double* x, fkt_cg_diagnostics* diag) {
  return guarded([&] {
    auto k = spec(kernel, keys, values, nparams);
    if (!(tolerance > 0.0)) throw std::invalid_argument("cgSolve requires a positive tolerance");
    requireDevice();
    cudaStream_t st;
    FKTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      fktb::DeviceNoisyOperator op;
      fktb::setupDenseOperator(op, n, d, points, k, has_diagonal != 0, diagonal, st);
      op.kernelDiagonal = fktb::safeKernelDiagonal(k, has_diagonal != 0, diagonal);
      const size_t bytes = static_cast<size_t>(n) * sizeof(double);
      op.noise.resize(static_cast<size_t>(n));
      fktb::DeviceBuffer<double> dRhs(static_cast<size_t>(n)), dX(static_cast<size_t>(n));
      FKTB_CUDA(cudaMemcpyAsync(op.noise.get(), noise, bytes, cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dRhs.get(), rhs, bytes, cudaMemcpyHostToDevice, st));
      const auto dg = fktb::cgSolveDevice(op, dRhs.get(), tolerance, max_iterations, jacobi != 0, dX.get(), st,
                                          restart_on_increase != 0);
      FKTB_CUDA(cudaMemcpyAsync(x, dX.get(), bytes, cudaMemcpyDeviceToHost, st));
      FKTB_CUDA(cudaStreamSynchronize(st));
      toC(dg, diag);
    } catch (...) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
  });
}

int fkt_gp_posterior_mean(int n_train, int d, const double* train_x, const double* y, const double* noise,
                          const char* kernel, const char* const* keys, const double* values, int nparams, int n_test,
                          const double* test_x, const fkt_gp_options* opt, double* mean, fkt_cg_diagnostics* diag) {
  return guarded([&] {
    auto k = spec(kernel, keys, values, nparams);
    fkt_gp_options def;
    fkt_default_gp_options(&def);
    const fkt_gp_options& o = opt ? *opt : def;
    fktb::GpDeviceOptions go;
    go.fkt = toPlanOptions(&o.fkt);
    go.cgTolerance = o.cg_tolerance;
    go.cgMaxIterations = o.cg_max_iterations;
    go.jacobi = o.jacobi != 0;
    go.dense = o.dense != 0;
    go.hasPriorMean = o.has_prior_mean != 0;
    go.priorMean = o.prior_mean;
    go.restartOnIncrease = o.restart_on_increase != 0;
    if (n_train < 1) throw std::invalid_argument("point cloud must be nonempty");
    if (n_test < 0) throw DimensionMismatch("gpPosteriorMean: negative test size");
    requireDevice();
    toC(fktb::gpPosteriorMeanGpu(n_train, d, train_x, y, noise, k, n_test, test_x, go, mean), diag);
  });
}

int fkt_plan_near_forms(fkt_plan_t plan, long long* gram_tiles, long long* total_tiles) {
  return guarded([&] {
    if (!plan || !gram_tiles || !total_tiles) throw std::invalid_argument("null argument");
    *gram_tiles = fktb::nearGramTiles(*plan->plan);
    *total_tiles = static_cast<long long>(plan->plan->nearTilesHost.size());
  });
}

long long fkt_plan_kernel_launches(fkt_plan_t plan, int nrhs) {
  long long out = -1;
  guarded([&] { out = fktb::kernelLaunches(*plan->plan, std::max(1, nrhs)); });
  return out;
}

int fkt_shard_cuts(const uint32_t* leaf_end, const unsigned long long* leaf_cum_cost, int leaves, int shards, uint32_t n,
                   uint32_t* cuts) {
  return guarded([&] {
    if (shards < 1 || leaves < 0) throw std::invalid_argument("shard_cuts: shards >= 1, leaves >= 0");
    std::vector<std::pair<uint32_t, unsigned long long>> le(static_cast<size_t>(leaves));
    for (int i = 0; i < leaves; ++i) le[static_cast<size_t>(i)] = {leaf_end[i], leaf_cum_cost[i]};
    const auto c = fktb::shardCutsFromLeaves(le, shards, n);
    std::copy(c.begin(), c.end(), cuts);
  });
}

fkt_tree_t fkt_plan_tree(fkt_plan_t plan) {
  // Borrowed view owned by the plan handle (freed with it).
  std::lock_guard<std::mutex> lock(plan->viewMutex);
  if (!plan->view || plan->view->tree != plan->plan->tree.get()) {
    plan->view = std::make_unique<fkt_tree_s>();
    plan->view->tree = plan->plan->tree.get();
  }
  return plan->view.get();
}

int fkt_tree_create(int n, int d, const double* x, int leaf_capacity, fkt_tree_t* out) {
  *out = nullptr;
  return guarded([&] {
    if (leaf_capacity < 1) throw std::invalid_argument("leaf capacity must be >= 1");
    if (n < 1) throw std::invalid_argument("point cloud must be nonempty");
    requireDevice();
    auto h = std::make_unique<fkt_tree_s>();
    FKTB_CUDA(cudaStreamCreateWithFlags(&h->ownedStream, cudaStreamNonBlocking));
    h->owned = std::make_unique<fktb::DeviceTree>();
    fktb::buildTreeGpu(*h->owned, x, n, d, leaf_capacity, h->ownedStream);
    h->tree = h->owned.get();
    *out = h.release();
  });
}

int fkt_tree_compute_sets(fkt_tree_t tree, double theta) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(tree->mutex);
    fktb::computeSetsGpu(*tree->tree, theta);
    tree->farReady = tree->nearReady = false;
  });
}

int fkt_tree_destroy(fkt_tree_t tree) {
  return guarded([&] {
    if (!tree || !tree->owned) return;  // borrowed views die with their plan
    cudaStream_t st = tree->ownedStream;
    tree->owned.reset();
    delete tree;
    if (st) cudaStreamDestroy(st);
  });
}

int fkt_tree_sizes(fkt_tree_t tree, long long* nodes, long long* depth, long long* far_total, long long* near_total,
                   double* theta) {
  return guarded([&] {
    const auto& t = *tree->tree;
    if (nodes) *nodes = t.nodes;
    if (depth) *depth = t.depth;
    if (far_total) *far_total = t.hasSets ? t.farTotal : 0;
    if (near_total) *near_total = t.hasSets ? t.nearTotal : 0;
    if (theta) *theta = t.hasSets ? t.theta : 0.0;
  });
}

int fkt_tree_nodes(fkt_tree_t tree, uint32_t* begin, uint32_t* end, int* left, int* right, double* radius,
                   double* center, double* box_lo, double* box_hi) {
  return guarded([&] {
    const auto& t = *tree->tree;
    const size_t nn = static_cast<size_t>(t.nodes), nd = nn * t.d;
    if (begin) std::memcpy(begin, t.begin.data(), nn * sizeof(uint32_t));
    if (end) std::memcpy(end, t.end.data(), nn * sizeof(uint32_t));
    if (left) std::memcpy(left, t.left.data(), nn * sizeof(int));
    if (right) std::memcpy(right, t.right.data(), nn * sizeof(int));
    if (radius) std::memcpy(radius, t.radius.data(), nn * sizeof(double));
    if (center) std::memcpy(center, t.center.data(), nd * sizeof(double));
    if (box_lo) std::memcpy(box_lo, t.boxLo.data(), nd * sizeof(double));
    if (box_hi) std::memcpy(box_hi, t.boxHi.data(), nd * sizeof(double));
  });
}

int fkt_tree_order(fkt_tree_t tree, uint32_t* order) {
  return guarded([&] {
    const auto& t = *tree->tree;
    FKTB_CUDA(cudaMemcpy(order, t.order.get(), t.order.bytes(), cudaMemcpyDeviceToHost));
  });
}

int fkt_tree_points(fkt_tree_t tree, double* perm) {
  return guarded([&] {
    const auto& t = *tree->tree;
    std::vector<double> soa(static_cast<size_t>(t.n) * t.d);
    FKTB_CUDA(cudaMemcpy(soa.data(), t.pc.get(), t.pc.bytes(), cudaMemcpyDeviceToHost));
    for (int pos = 0; pos < t.n; ++pos)
      for (int a = 0; a < t.d; ++a) perm[static_cast<size_t>(pos) * t.d + a] = soa[static_cast<size_t>(a) * t.n + pos];
  });
}

static int treeSets(fkt_tree_t tree, bool far, long long* off, uint32_t* idx) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(tree->mutex);
    const auto& t = *tree->tree;
    if (!t.hasSets) throw std::invalid_argument("interaction sets not computed");
    bool& ready = far ? tree->farReady : tree->nearReady;
    auto& o = far ? tree->farOff : tree->nearOff;
    auto& v = far ? tree->farIdx : tree->nearIdx;
    if (!ready) {
      fktb::materializeSets(t, far, o, v);
      ready = true;
    }
    if (off) std::memcpy(off, o.data(), o.size() * sizeof(long long));
    if (idx) std::memcpy(idx, v.data(), v.size() * sizeof(uint32_t));
  });
}

int fkt_tree_far_sets(fkt_tree_t tree, long long* off, uint32_t* idx) { return treeSets(tree, true, off, idx); }
int fkt_tree_near_sets(fkt_tree_t tree, long long* off, uint32_t* idx) { return treeSets(tree, false, off, idx); }

int fkt_dense_rows(int n, int d, const double* x, const char* kernel, const char* const* keys, const double* values,
                   int nparams, const double* y, int m, const int64_t* rows, double* z, int has_diagonal,
                   double diagonal) {
  return guarded([&] {
    auto k = spec(kernel, keys, values, nparams);
    if (d < 1 || d > FKTB_MAX_DIM) throw Unsupported("unsupported on the GPU path: dense rows need 1 <= d <= 16");
    for (int i = 0; i < m; ++i)
      if (rows[i] < 0 || rows[i] >= n) throw std::invalid_argument("dense rows: row index out of range");
    requireDevice();
    FktbKernelDesc kd;
    fktb::fillKernelDesc(k, kd);
    if (has_diagonal)
      kd.diag = diagonal;
    else if (!k.valueAtZero)
      throw std::domain_error("kernel '" + k.name + "' is singular at r = 0 and no diagonal convention is set");
    cudaStream_t st;
    FKTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    {
      fktb::DeviceBuffer<double> dx(static_cast<size_t>(n) * d), dy(static_cast<size_t>(n)), dz(static_cast<size_t>(std::max(m, 1)));
      fktb::DeviceBuffer<int64_t> dr(static_cast<size_t>(std::max(m, 1)));
      FKTB_CUDA(cudaMemcpyAsync(dx.get(), x, dx.bytes(), cudaMemcpyHostToDevice, st));
      FKTB_CUDA(cudaMemcpyAsync(dy.get(), y, dy.bytes(), cudaMemcpyHostToDevice, st));
      if (m > 0) FKTB_CUDA(cudaMemcpyAsync(dr.get(), rows, static_cast<size_t>(m) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      fktb::denseRowsGpu(n, d, dx.get(), kd, dy.get(), m, dr.get(), dz.get(), st);
      if (m > 0) FKTB_CUDA(cudaMemcpyAsync(z, dz.get(), static_cast<size_t>(m) * sizeof(double), cudaMemcpyDeviceToHost, st));
      FKTB_CUDA(cudaStreamSynchronize(st));
    }
    cudaStreamDestroy(st);
  });
}

int fkt_dense_multiply(int n, int d, const double* x, const char* kernel, const char* const* keys, const double* values,
                       int nparams, const double* y, double* z, int has_diagonal, double diagonal) {
  std::vector<int64_t> rows(static_cast<size_t>(std::max(n, 0)));
  for (int i = 0; i < n; ++i) rows[static_cast<size_t>(i)] = i;
  return fkt_dense_rows(n, d, x, kernel, keys, values, nparams, y, n, rows.data(), z, has_diagonal, diagonal);
}

int fkt_relative_error(const double* approx, const double* exact, long long n, double* out) {
  return guarded([&] {
    double num = 0.0, den = 0.0;
    for (long long i = 0; i < n; ++i) {
      const double diff = approx[i] - exact[i];
      num += diff * diff;
      den += exact[i] * exact[i];
    }
    if (den == 0.0) throw ZeroReference("relative error against a zero reference vector");
    *out = std::sqrt(num / den);
  });
}

long long fkt_expansion_size(int d, int p) {
  long long r = -1;
  guarded([&] { r = static_cast<long long>(fktb::expansionSize(d, p)); });
  return r;
}

int fkt_tbar(int d, int p, int k, int j, int m, double* value, char* exact, int exact_len) {
  return guarded([&] {
    if (p > fktb::kMaxExpansionOrder)
      throw OrderTooLarge("expansion order " + std::to_string(p) + " exceeds the supported cap " +
                          std::to_string(fktb::kMaxExpansionOrder));
    const auto& t = fktb::coefTable(d, p);
    const auto& q = t.tbar(k, j, m);
    if (value) *value = t.tbarDouble(k, j, m);
    if (exact && exact_len > 0) {
      std::string s = q.num().str() + "/" + q.den().str();
      std::strncpy(exact, s.c_str(), static_cast<size_t>(exact_len) - 1);
      exact[exact_len - 1] = 0;
    }
  });
}

long long fkt_tbar_serialize(int d, int p, char* buf, long long len) {
  long long need = -1;
  guarded([&] {
    if (p > fktb::kMaxExpansionOrder)
      throw OrderTooLarge("expansion order " + std::to_string(p) + " exceeds the supported cap " +
                          std::to_string(fktb::kMaxExpansionOrder));
    const std::string s = fktb::coefTable(d, p).serialize();
    need = static_cast<long long>(s.size()) + 1;
    if (buf && len > 0) {
      const size_t n = static_cast<size_t>(std::min<long long>(len - 1, static_cast<long long>(s.size())));
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
  return need;
}

int fkt_tbar_deserialize(const char* text, int* d, int* p, int* equals_computed) {
  return guarded([&] {
    auto t = fktb::CoefTable::deserialize(text ? std::string(text) : std::string());
    if (!t) throw std::invalid_argument("coefficient table text does not parse");
    *d = t->dimension();
    *p = t->maxOrder();
    if (equals_computed) *equals_computed = t->maxOrder() <= fktb::kMaxExpansionOrder &&
                                            *t == fktb::coefTable(t->dimension(), t->maxOrder());
  });
}

int fkt_compression_ranks(const char* kernel, const char* const* keys, const double* values, int nparams, int d, int p,
                          int* ranks) {
  return guarded([&] {
    auto k = spec(kernel, keys, values, nparams);
    if (p > fktb::kMaxExpansionOrder)
      throw OrderTooLarge("expansion order " + std::to_string(p) + " exceeds the supported cap " +
                          std::to_string(fktb::kMaxExpansionOrder));
    auto f = fktb::radialCompression(k, fktb::coefTable(d, p), p);
    for (int i = 0; i <= p; ++i) ranks[i] = f[static_cast<size_t>(i)].rank;
  });
}

double fkt_addition_normalizer(int d, int k) {
  double r = 0.0;
  guarded([&] { r = fktb::additionNormalizer(d, k); });
  return r;
}

long long fkt_harmonic_count(int d, int k) {
  long long r = -1;
  guarded([&] { r = static_cast<long long>(fktb::harmonicIndexCount(d, k)); });
  return r;
}

int fkt_synth_cloud(const char* kind, int n, int d, uint64_t seed, double* x, double* y) {
  return guarded([&] { fktb::synthCloud(kind, n, d, seed, x, y); });
}

int fkt_synth_config(int cfg, int n, uint64_t seed, double* x, double* w) {
  return guarded([&] { fktb::synthConfig(cfg, n, seed, x, w); });
}

int fkt_config_dims(int cfg, int* d, int* nrhs) { return fktb::configDims(cfg, d, nrhs); }

}  // extern "C"
