/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference FKT hot
 * path (checker for the CUDA product; see fkt_oracle.c for the reference
 * file:line each function follows). Loaded by tests/ through ctypes
 * (oracle/restated.py). Never linked into the product. */
#ifndef FKT_ORACLE_H
#define FKT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fko_tree fko_tree;

fko_tree* fko_tree_build(int n, int d, const double* x, int leaf);
void fko_tree_free(fko_tree* t);
int fko_tree_node_count(const fko_tree* t);
void fko_tree_arrays(const fko_tree* t, uint32_t* order, uint32_t* begin, uint32_t* end, int* left, int* right,
                     double* radius, double* center, double* box_lo, double* box_hi, double* perm);
int fko_tree_sets(fko_tree* t, double theta, long long* far_total, long long* near_total);
void fko_tree_set_arrays(const fko_tree* t, long long* far_off, uint32_t* far, long long* near_off, uint32_t* near);

void fko_fingerprints(int n, const uint32_t* order, int nodes, const long long* far_off, const uint32_t* far,
                      const long long* near_off, const uint32_t* near, const double* radius, const double* center,
                      int d, uint64_t out[3]);

/* prm = {s2, a, is2, rho} */
double fko_kernel(int id, const double* prm, double r);
void fko_kernel_jet(int id, const double* prm, double r, int p, double* c);

typedef struct fko_tables {
  int d, p;
  const double* tbar;        /* (p+1)^3, index (k*(p+1)+j)*(p+1)+m */
  int H;                     /* harmonics of degree <= p */
  const int* hdeg;           /* H */
  const int* chain_m;        /* H x (d-1): m0 = k, m1.. (abs values) */
  const int* chain_phase;    /* H */
  const double* chain_norm;  /* H */
  const double* zk;          /* p+1 */
  int compressed;
  const int* ranks;          /* p+1 */
  const int* tgt_off;        /* nf+1, factors ordered by (k, i) */
  const int* tgt_pow;
  const double* tgt_c;
  const int* src_off;
  const int* src_pow;
  const double* src_c;
} fko_tables;

/* z = K y (streaming operators), threads <= 0 -> all */
int fko_multiply(const fko_tree* t, int kernel_id, const double* prm, double diag, const fko_tables* tab,
                 const double* y, double* z, int threads);

int fko_dense_rows(int n, int d, const double* x, int kernel_id, const double* prm, double diag, const double* y,
                   int m, const int64_t* rows, double* z, int threads);

#ifdef __cplusplus
}
#endif

#endif
