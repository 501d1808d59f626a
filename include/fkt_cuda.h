/*
 * fkt_cuda.h — C-ABI of the B200-native Fast Kernel Transform MVM.
 *
 * Plain C: opaque handles, pointers and sizes, int status codes and a
 * thread-local message (no C++ exceptions cross this boundary). The C++
 * operator API in include/fkt/*.hpp (a drop-in for the reference's
 * proj/include/fkt) and the Python mirror (paper_2106_04487_b200) are thin
 * layers over these entry points; see INTEGRATION.md.
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef FKT_CUDA_H
#define FKT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; each maps to a reference exception type. */
enum {
  FKT_OK = 0,
  FKT_ERR_INVALID_ARGUMENT = 1,   /* std::invalid_argument */
  FKT_ERR_DIMENSION_MISMATCH = 2, /* fkt::DimensionMismatchError (transform.hpp:17-20) */
  FKT_ERR_ORDER_TOO_LARGE = 3,    /* fkt::OrderTooLargeError (coefficients.hpp:23-28) */
  FKT_ERR_NOT_RECURRENCE = 4,     /* fkt::NotRecurrenceKernelError (expansion.hpp:27-31) */
  FKT_ERR_SINGULAR_AT_ZERO = 5,   /* fkt::SingularAtZeroError (kernels.hpp:22-26) */
  FKT_ERR_ZERO_REFERENCE = 6,     /* fkt::ZeroReferenceError (transform.hpp:22-25) */
  FKT_ERR_CUDA = 7,               /* device failure (no CPU fallback exists) */
  FKT_ERR_UNSUPPORTED = 8,        /* valid for the reference, not offered on the GPU path */
  FKT_ERR_INTERNAL = 9
};

/* Compression modes, reference transform.hpp:27. */
enum { FKT_COMPRESSION_AUTO = 0, FKT_COMPRESSION_ON = 1, FKT_COMPRESSION_OFF = 2 };

/* Reference fkt::FktOptions (transform.hpp:29-41). */
typedef struct fkt_options {
  int p;
  double theta;
  int leaf_capacity;
  int compression;
  int eager_operators; /* accepted; the GPU always recomputes operators in registers */
  int barnes_hut;      /* Barnes-Hut monopole far field (transform.cpp:44-60,131-146); forces p = 0 */
  int threads;         /* CPU-only knob, ignored */
  int has_diagonal;
  double diagonal;
  int near_precision;  /* additive extension: 64 (default, FP64) or 32 (FP32 fast near field) */
  int deterministic;   /* additive extension: 1 = bitwise reproducible z (fixed-order sums, no
                          atomics into z or the moments); the reference merges
                          its per-thread buffers in a fixed order (transform.cpp:194-203) */
} fkt_options;

typedef struct fkt_plan_s* fkt_plan_t;
typedef struct fkt_tree_s* fkt_tree_t;

typedef struct fkt_plan_info {
  int n, d, p;
  long long nodes, leaves, depth;
  long long far_total, near_total;
  long long coefficient_count; /* reference FktPlan::coefficientCount() */
  long long stored_coefficients;
  int compressed;              /* reference FktPlan::compressed() */
  double plan_seconds;
  long long far_tiles, near_tiles, s2m_tiles;
  int m2t_cartesian;           /* 1: single-RHS multiplies run the Cartesian (q-form) M2T */
} fkt_plan_info;

/* Last error message / code of the calling thread. */
const char* fkt_last_error(void);
int fkt_last_error_code(void);

/* Library version string and the 14 built-in kernel names
 * (reference builtinKernelNames(), kernels.hpp:85). */
const char* fkt_version(void);
int fkt_kernel_count(void);
const char* fkt_kernel_name(int i);

/* Kernel validation and host evaluation (reference makeKernel, kernels.hpp:83,
 * IsotropicKernel::operator(), kernels.hpp:49-58). Parameters are parallel
 * key/value arrays. */
int fkt_kernel_check(const char* name, const char* const* keys, const double* values, int nparams,
                     int* has_recurrence, int* has_value_at_zero, double* value_at_zero);
int fkt_kernel_eval(const char* name, const char* const* keys, const double* values, int nparams,
                    const double* r, double* out, long long count, int has_diagonal, double diagonal);

/* The registered derivative recurrence K' = q K of a built-in kernel
 * (kernels.hpp:68, kernels.cpp:37-156) as exact rational Laurent terms: writes
 * up to max_terms (power, "num/den") pairs, text NUL-separated into buf of
 * buf_len bytes; *terms = the count (0 and FKT_OK when the kernel has none). */
int fkt_kernel_recurrence(const char* name, const char* const* keys, const double* values, int nparams, int* terms,
                          int* powers, int max_terms, char* buf, long long buf_len);

/* K on a jet argument (kernels.hpp:61-66): in = coefficients c_0..c_order of
 * the argument series at `center`, out = those of K(argument). */
int fkt_kernel_eval_jet(const char* name, const char* const* keys, const double* values, int nparams, double center,
                        int order, const double* in, double* out);

void fkt_default_options(fkt_options* opt);

/* fkt::FktPlan(PointCloud, KernelPtr, FktOptions) — transform.cpp:39-92.
 * x: host, row-major n x d. */
int fkt_plan_create(int n, int d, const double* x, const char* kernel, const char* const* keys,
                    const double* values, int nparams, const fkt_options* opt, fkt_plan_t* out);
int fkt_plan_destroy(fkt_plan_t plan);
/* Additive (no reference counterpart; the reference rebuilds FktPlan from a
 * new PointCloud, transform.cpp:39-92): the same plan on new coordinates of
 * the same n points, x host row-major n x d. Tree, interaction sets, tiles and
 * moment plan are rebuilt on the GPU reusing the plan's buffers; the result
 * equals fkt_plan_create on x with the plan's kernel and options. Cached plans
 * (fkt_plan_cache_get) are shared and refuse it. */
int fkt_plan_rebuild(fkt_plan_t plan, const double* x);
/* The same with the new coordinates already in device memory (row-major
 * n x d, FP64; e.g. a t-SNE embedding updated on the GPU): no host copy. The
 * caller's writes to x_dev must have completed (or be ordered before the
 * plan's work by a device synchronisation); returns once the plan is rebuilt. */
int fkt_plan_rebuild_device(fkt_plan_t plan, const double* x_dev);
int fkt_plan_info_get(fkt_plan_t plan, fkt_plan_info* info);

/* Plan cache (the reference rebuilds a plan per call site, e.g.
 * gp.cpp:148-151, 162-168). Returns a plan for (x, kernel, options), built
 * only when no identical plan (same coordinates bytewise, kernel, parameters
 * and options) is cached; *hit tells which. Every get must be paired with a
 * release (fkt_plan_destroy refuses cached plans). Unreferenced plans stay
 * cached up to the capacity (default 4) and are evicted least recently used
 * first. Cached plans are shared: do not fkt_plan_set_shard them. */
int fkt_plan_cache_get(int n, int d, const double* x, const char* kernel, const char* const* keys,
                       const double* values, int nparams, const fkt_options* opt, fkt_plan_t* out, int* hit);
int fkt_plan_cache_release(fkt_plan_t plan);
int fkt_plan_cache_set_capacity(int plans);
int fkt_plan_cache_size(void);

/* fkt::FktPlan::multiply(span y) — transform.cpp:184-204. Host buffers,
 * synchronous; nrhs column-major right-hand sides (length n*nrhs). */
int fkt_plan_multiply(fkt_plan_t plan, const double* y, double* z, int nrhs);
/* Same on device buffers, enqueued on `stream` (cudaStream_t; NULL = the
 * plan's own stream, synchronised before return). */
int fkt_plan_multiply_device(fkt_plan_t plan, const double* y_dev, double* z_dev, int nrhs, void* stream);
/* Stage-level device calls used by the benchmark to time kernels. stage:
 * 0 gather, 1 s2m, 2 near, 3 m2t, 4 scatter (workspaces owned by the plan). */
int fkt_plan_stage_device(fkt_plan_t plan, int stage, const double* y_dev, double* z_dev, int nrhs, void* stream);

/* Multi-GPU target sharding (replaces the node-chunked thread
 * split of FktPlan::multiply, transform.cpp:18-35,184-204). Every rank holds
 * the full plan and owns the contiguous, cost-balanced range
 * [pos_lo, pos_hi) of tree positions. Under a shard, multiply computes
 *   stage 1: partial node moments from the owned sources only,
 *   stage 2/3: near and far interactions of the owned targets only,
 * so z is exact on the owned targets and 0 elsewhere PROVIDED the moment
 * tables were summed over all ranks between stages 1 and 3 (the one data-path
 * exchange; fkt_plan_moments_device exposes the table, [rhs][node][P], count =
 * nodes * P per right-hand side). shards = 1 restores the whole problem. */
int fkt_plan_set_shard(fkt_plan_t plan, int shard, int shards);
/* The whole sharded MVM in one call (csrc/multigpu.cu): gather, S2M of the
 * owned sources, NCCL all-reduce of the moments, near + M2T of the owned
 * targets, NCCL broadcast of every rank's owned z range, scatter -- all of z
 * on every rank, captured as one CUDA graph per (y, z, nrhs, stream). The plan
 * must be set to shard (rank, size) of the communicator. nccl_comm: an
 * ncclComm_t, e.g. from fkt_nccl_comm_create; NCCL is loaded at run time
 * (libnccl.so.2), FKT_ERR_UNSUPPORTED when it is not loadable. */
int fkt_plan_multiply_sharded(fkt_plan_t plan, const double* y_dev, double* z_dev, int nrhs, void* nccl_comm,
                              void* stream);
/* NCCL communicator helpers: rank 0 makes a 128-byte id, every rank passes it
 * (shared over any side channel, e.g. torch.distributed) to comm_create. */
int fkt_nccl_unique_id(char* id128);
int fkt_nccl_comm_create(const char* id128, int nranks, int rank, void** comm);
int fkt_nccl_comm_destroy(void* comm);
int fkt_plan_shard_range(fkt_plan_t plan, long long* pos_lo, long long* pos_hi);
int fkt_plan_moments_device(fkt_plan_t plan, double** moments, long long* count_per_rhs);
/* Near-field tiles (leaf, <= 256 targets) of the FP64 near field, and how many
 * of them run the Gram pair form (leaf-centred |t|^2 + |s|^2 - 2 t.s; DESIGN.md
 * §3) instead of the difference form. No reference counterpart (diagnostic). */
int fkt_plan_near_forms(fkt_plan_t plan, long long* gram_tiles, long long* total_tiles);
/* How many of this library's kernels one multiply with nrhs right-hand sides
 * launches on the current shard (memsets excluded); -1 on error. */
long long fkt_plan_kernel_launches(fkt_plan_t plan, int nrhs);
/* The cut rule (host only): leaves in position order with their end position
 * and cumulative cost; cuts has shards+1 entries (cuts[0]=0, cuts[shards]=n). */
int fkt_shard_cuts(const uint32_t* leaf_end, const unsigned long long* leaf_cum_cost, int leaves, int shards, uint32_t n,
                   uint32_t* cuts);

/* Gaussian-process solves (reference proj/include/fkt/gp.hpp, gp.cpp). The
 * CG iterates stay in HBM (x, r, z, p, Ap); each iteration is one device MVM
 * plus small vector kernels, the host reads two scalars per iteration. */
typedef struct fkt_cg_diagnostics { /* CgDiagnostics, gp.hpp:35-40 */
  int iterations;
  double final_residual; /* relative to |b| */
  int converged;
  int restarts;
} fkt_cg_diagnostics;

/* cgSolve(NoisyOperator(plan, noise), rhs, ...) — gp.cpp:20-26, 58-124.
 * Host buffers of length n. restart_on_increase = 1 is the reference's rule
 * (restart from the current iterate whenever |r| grows, gp.cpp:100-111);
 * 0 (additive) runs textbook CG. */
int fkt_cg_solve(fkt_plan_t plan, const double* noise, const double* rhs, double tolerance, int max_iterations,
                 int jacobi, int restart_on_increase, double* x, fkt_cg_diagnostics* diag);
/* The same over the dense operator NoisyOperator(cloud, kernel, noise,
 * diagonal) — gp.cpp:28-37 (K7 rows on the GPU). */
int fkt_cg_solve_dense(int n, int d, const double* points, const char* kernel, const char* const* keys,
                       const double* values, int nparams, int has_diagonal, double diagonal, const double* noise,
                       const double* rhs, double tolerance, int max_iterations, int jacobi, int restart_on_increase,
                       double* x, fkt_cg_diagnostics* diag);

typedef struct fkt_gp_options { /* GpOptions, gp.hpp:51-58 */
  fkt_options fkt;
  double cg_tolerance;
  int cg_max_iterations;
  int jacobi;
  int dense;
  int has_prior_mean;
  double prior_mean;
  int restart_on_increase; /* additive; 1 = the reference's CG restart rule (default) */
} fkt_gp_options;
void fkt_default_gp_options(fkt_gp_options* opt);

/* gpPosteriorMean(train, y, noise, kernel, test, options) — gp.cpp:126-177:
 * CG on the train plan, then one multiply on the concatenated train+test
 * cloud with the solution zero-padded on the test block. mean: n_test. */
int fkt_gp_posterior_mean(int n_train, int d, const double* train_x, const double* y, const double* noise,
                          const char* kernel, const char* const* keys, const double* values, int nparams, int n_test,
                          const double* test_x, const fkt_gp_options* opt, double* mean, fkt_cg_diagnostics* diag);

/* Tree view of a plan (borrowed; valid while the plan lives). */
fkt_tree_t fkt_plan_tree(fkt_plan_t plan);

/* fkt::PartitionTree(cloud, leafCapacity) + computeInteractionSets(theta) —
 * tree.hpp:43-79, tree.cpp:29-213. Built on the GPU. */
int fkt_tree_create(int n, int d, const double* x, int leaf_capacity, fkt_tree_t* out);
int fkt_tree_compute_sets(fkt_tree_t tree, double theta);
int fkt_tree_destroy(fkt_tree_t tree);
/* nodes, depth, far/near totals (0 before computeInteractionSets), theta */
int fkt_tree_sizes(fkt_tree_t tree, long long* nodes, long long* depth, long long* far_total,
                   long long* near_total, double* theta);
/* Node arrays in reference pre-order (tree.hpp:30-41); any pointer may be NULL.
 * center/box_lo/box_hi: nodes x d. */
int fkt_tree_nodes(fkt_tree_t tree, uint32_t* begin, uint32_t* end, int* left, int* right, double* radius,
                   double* center, double* box_lo, double* box_hi);
/* PartitionTree::order() (permuted position -> original index) and the
 * permuted coordinates pointAt(pos) (n x d row-major). */
int fkt_tree_order(fkt_tree_t tree, uint32_t* order);
int fkt_tree_points(fkt_tree_t tree, double* perm);
/* farSet / nearSet of every node as CSR of ORIGINAL indices, ascending
 * (tree.hpp:37-38); off has nodes+1 entries. */
int fkt_tree_far_sets(fkt_tree_t tree, long long* off, uint32_t* idx);
int fkt_tree_near_sets(fkt_tree_t tree, long long* off, uint32_t* idx);

/* fkt::denseMultiply (transform.cpp:210-237) on the GPU, and a sampled-row
 * variant (rows: original indices). Host buffers. */
int fkt_dense_multiply(int n, int d, const double* x, const char* kernel, const char* const* keys,
                       const double* values, int nparams, const double* y, double* z, int has_diagonal,
                       double diagonal);
int fkt_dense_rows(int n, int d, const double* x, const char* kernel, const char* const* keys,
                   const double* values, int nparams, const double* y, int m, const int64_t* rows,
                   double* z, int has_diagonal, double diagonal);

/* fkt::relativeError (transform.cpp:245-255). */
int fkt_relative_error(const double* approx, const double* exact, long long n, double* out);

/* fkt::expansionSize (expansion.hpp:34): binom(d+p, p). */
long long fkt_expansion_size(int d, int p);

/* Plan-time expansion tables (host, no GPU needed): exact T-bar_kjm
 * (coefficients.hpp:47-52) as a double and as "num/den" text; the exact
 * compression ranks per degree (expansion.cpp:190-243; -1 entries when the
 * kernel has no recurrence -> FKT_ERR_NOT_RECURRENCE); Z_k
 * (harmonics.hpp:56). */
int fkt_tbar(int d, int p, int k, int j, int m, double* value, char* exact, int exact_len);
/* CoefficientTable::serialize (coefficients.cpp:113-124): the exact T-bar
 * table as text. Writes at most len bytes (NUL-terminated when len > 0) and
 * returns the length needed including the NUL, -1 on error. Every plan also
 * honours the reference's FKT_CACHE_DIR cache in this format. */
long long fkt_tbar_serialize(int d, int p, char* buf, long long len);
/* CoefficientTable::deserialize (:126-166): FKT_ERR_INVALID_ARGUMENT when the
 * text does not parse (the reference returns nullopt); else d, p and whether
 * the table equals the one computed here (operator==, :168-170). */
int fkt_tbar_deserialize(const char* text, int* d, int* p, int* equals_computed);
int fkt_compression_ranks(const char* kernel, const char* const* keys, const double* values, int nparams, int d,
                          int p, int* ranks);
double fkt_addition_normalizer(int d, int k);
long long fkt_harmonic_count(int d, int k);

/* Plan-time phases in seconds, in this order: tree (K1), interaction sets
 * (K2), exact tables, work tiles, near-field geometry rows, moment plan,
 * other (workspaces, drains). Writes min(count, 7) values. */
int fkt_plan_phases(fkt_plan_t plan, double* seconds, int count);

/* Measurement support: FMA-pipe peak (FLOP/s, FMA = 2) of the current device,
 * fp64 (fp32 = 0) or fp32 (fp32 = 1): the roofline denominator for the
 * FP64-bound kernels. */
int fkt_fma_peak(int fp32, double* flops_per_s);
/* The two FP64 probes behind fkt_fma_peak(0): DFMA chains and FP64 tensor-core
 * (mma.sync m8n8k4) chains; they share one datapath on B200. */
int fkt_fp64_peaks(double* dfma_flops_per_s, double* dmma_flops_per_s);

/* Seeded synthetic inputs (reference fkt::Rng, synthetic.hpp:17-50;
 * generators synthetic.cpp:7-55). kind: "cube", "sphere", "mixture".
 * y (optional) receives normalVector(n) drawn after the cloud. */
int fkt_synth_cloud(const char* kind, int n, int d, uint64_t seed, double* x, double* y);
/* The five BASELINE configurations (SURVEY Appendix B recipes). */
int fkt_synth_config(int cfg, int n, uint64_t seed, double* x, double* w);
int fkt_config_dims(int cfg, int* d, int* nrhs);

#ifdef __cplusplus
}
#endif

#endif /* FKT_CUDA_H */
