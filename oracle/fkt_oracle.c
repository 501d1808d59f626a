/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference FKT hot
 * path, the CPU checker for the CUDA product (never linked into it).
 * Pinned against the reference itself (oracle/_ref, tests/golden fixtures)
 * by tests/test_oracle.py. Reference citations are proj/... file:line.
 * Built with -ffp-contract=off so the tree geometry is bit-identical. */
#include "fkt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Tree: proj/src/tree.cpp:13-171 */

typedef struct {
  uint32_t begin, end;
  int left, right;
  double radius;
  double* lo; /* d */
  double* hi;
  double* c;
} fko_node;

struct fko_tree {
  int n, d, leaf;
  uint32_t* order;
  double* perm;
  fko_node* nodes;
  int count, cap;
  double theta;
  long long *far_off, *near_off;
  uint32_t *far, *near;
  long long far_total, near_total;
};

/* tree.cpp:13-25 */
static void regularize(double* lo, double* hi, int d) {
  double maxSide = 0.0;
  for (int a = 0; a < d; ++a) {
    const double s = hi[a] - lo[a];
    if (maxSide < s) maxSide = s;
  }
  if (maxSide <= 0.0) return;
  for (int a = 0; a < d; ++a) {
    const double side = hi[a] - lo[a];
    if (side < 0.5 * maxSide) {
      const double pad = 0.5 * (0.5 * maxSide - side);
      lo[a] -= pad;
      hi[a] += pad;
    }
  }
}

/* k-th smallest (quickselect on a copy): the value std::nth_element puts at k */
static double select_kth(double* v, size_t n, size_t k) {
  size_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const double pivot = v[lo + (hi - lo) / 2];
    size_t i = lo, j = hi;
    while (i <= j) {
      while (v[i] < pivot) ++i;
      while (pivot < v[j]) --j;
      if (i <= j) {
        const double t = v[i];
        v[i] = v[j];
        v[j] = t;
        ++i;
        if (j == 0) break;
        --j;
      }
    }
    if (k <= j)
      hi = j;
    else if (k >= i)
      lo = i;
    else
      return v[k];
  }
  return v[k];
}

static int push_node(fko_tree* t) {
  if (t->count == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 64;
    t->nodes = (fko_node*)realloc(t->nodes, (size_t)t->cap * sizeof(fko_node));
  }
  fko_node* nd = &t->nodes[t->count];
  memset(nd, 0, sizeof(*nd));
  nd->lo = (double*)malloc((size_t)t->d * sizeof(double));
  nd->hi = (double*)malloc((size_t)t->d * sizeof(double));
  nd->c = (double*)malloc((size_t)t->d * sizeof(double));
  nd->left = nd->right = -1;
  return t->count++;
}

/* tree.cpp:41-171 */
static int build_node(fko_tree* t, uint32_t b, uint32_t e, uint32_t* tmpIdx, double* tmpPts, double* vals) {
  const int d = t->d;
  const int idx = push_node(t);
  fko_node* nd = &t->nodes[idx];
  nd->begin = b;
  nd->end = e;
  for (int a = 0; a < d; ++a) {
    nd->lo[a] = INFINITY;
    nd->hi[a] = -INFINITY;
  }
  for (uint32_t pos = b; pos < e; ++pos) {
    const double* pt = t->perm + (size_t)pos * d;
    for (int a = 0; a < d; ++a) {
      if (pt[a] < nd->lo[a]) nd->lo[a] = pt[a];
      if (nd->hi[a] < pt[a]) nd->hi[a] = pt[a];
    }
  }
  double extent = 0.0;
  for (int a = 0; a < d; ++a) extent += nd->hi[a] - nd->lo[a];
  regularize(nd->lo, nd->hi, d);
  for (int a = 0; a < d; ++a) nd->c[a] = 0.5 * (nd->lo[a] + nd->hi[a]);
  double r2 = 0.0;
  for (uint32_t pos = b; pos < e; ++pos) {
    const double* pt = t->perm + (size_t)pos * d;
    double dist2 = 0.0;
    for (int a = 0; a < d; ++a) {
      const double q = pt[a] - nd->c[a];
      dist2 += q * q;
    }
    if (r2 < dist2) r2 = dist2;
  }
  nd->radius = sqrt(r2);
  if (e - b <= (uint32_t)t->leaf || extent == 0.0) return idx;

  int axis = 0;
  double best = -1.0;
  for (int a = 0; a < d; ++a) {
    const double side = nd->hi[a] - nd->lo[a];
    if (side > best) {
      best = side;
      axis = a;
    }
  }
  const double lo = nd->lo[axis], hi = nd->hi[axis];
  double maxOther = 0.0, minOther = INFINITY;
  for (int a = 0; a < d; ++a) {
    if (a == axis) continue;
    const double side = nd->hi[a] - nd->lo[a];
    if (maxOther < side) maxOther = side;
    if (side < minOther) minOther = side;
  }
  double cl = lo, ch = hi;
  if (d > 1) {
    const double c1 = lo + 0.5 * maxOther, c2 = hi - 2.0 * minOther;
    cl = c1 < c2 ? c2 : c1;
    const double c3 = lo + 2.0 * minOther, c4 = hi - 0.5 * maxOther;
    ch = c4 < c3 ? c4 : c3;
    if (cl > ch) cl = ch = 0.5 * (lo + hi);
  }
  const size_t cnt = e - b;
  for (size_t i = 0; i < cnt; ++i) vals[i] = t->perm[(size_t)(b + i) * d + axis];
  const double med = select_kth(vals, cnt, cnt / 2);
  double split = med < cl ? cl : (ch < med ? ch : med); /* std::clamp */

  size_t lower = 0;
  for (uint32_t pos = b; pos < e; ++pos) lower += t->perm[(size_t)pos * d + axis] <= split;
  if (lower == 0 || lower == cnt) { /* tree.cpp:136-159 */
    double mx = -INFINITY, below = -INFINITY;
    for (uint32_t pos = b; pos < e; ++pos) {
      const double v = t->perm[(size_t)pos * d + axis];
      if (mx < v) mx = v;
    }
    for (uint32_t pos = b; pos < e; ++pos) {
      const double v = t->perm[(size_t)pos * d + axis];
      if (v < mx && below < v) below = v;
    }
    split = below;
    lower = 0;
    for (uint32_t pos = b; pos < e; ++pos) lower += t->perm[(size_t)pos * d + axis] <= split;
  }
  size_t li = 0, ui = lower;
  for (uint32_t pos = b; pos < e; ++pos) {
    const double* pt = t->perm + (size_t)pos * d;
    const size_t dst = pt[axis] <= split ? li++ : ui++;
    tmpIdx[dst] = t->order[pos];
    memcpy(tmpPts + dst * d, pt, (size_t)d * sizeof(double));
  }
  memcpy(t->order + b, tmpIdx, cnt * sizeof(uint32_t));
  memcpy(t->perm + (size_t)b * d, tmpPts, cnt * d * sizeof(double));
  const uint32_t mid = b + (uint32_t)lower;
  const int l = build_node(t, b, mid, tmpIdx, tmpPts, vals);
  const int r = build_node(t, mid, e, tmpIdx, tmpPts, vals);
  t->nodes[idx].left = l;
  t->nodes[idx].right = r;
  return idx;
}

fko_tree* fko_tree_build(int n, int d, const double* x, int leaf) {
  if (n < 1 || leaf < 1 || d < 1) return NULL;
  fko_tree* t = (fko_tree*)calloc(1, sizeof(fko_tree));
  t->n = n;
  t->d = d;
  t->leaf = leaf;
  t->order = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  t->perm = (double*)malloc((size_t)n * d * sizeof(double));
  for (int i = 0; i < n; ++i) t->order[i] = (uint32_t)i;
  memcpy(t->perm, x, (size_t)n * d * sizeof(double));
  uint32_t* tmpIdx = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  double* tmpPts = (double*)malloc((size_t)n * d * sizeof(double));
  double* vals = (double*)malloc((size_t)n * sizeof(double));
  build_node(t, 0, (uint32_t)n, tmpIdx, tmpPts, vals);
  free(tmpIdx);
  free(tmpPts);
  free(vals);
  return t;
}

void fko_tree_free(fko_tree* t) {
  if (!t) return;
  for (int i = 0; i < t->count; ++i) {
    free(t->nodes[i].lo);
    free(t->nodes[i].hi);
    free(t->nodes[i].c);
  }
  free(t->nodes);
  free(t->order);
  free(t->perm);
  free(t->far_off);
  free(t->near_off);
  free(t->far);
  free(t->near);
  free(t);
}

int fko_tree_node_count(const fko_tree* t) { return t->count; }

void fko_tree_arrays(const fko_tree* t, uint32_t* order, uint32_t* begin, uint32_t* end, int* left, int* right,
                     double* radius, double* center, double* box_lo, double* box_hi, double* perm) {
  const int d = t->d;
  if (order) memcpy(order, t->order, (size_t)t->n * sizeof(uint32_t));
  if (perm) memcpy(perm, t->perm, (size_t)t->n * d * sizeof(double));
  for (int b = 0; b < t->count; ++b) {
    const fko_node* nd = &t->nodes[b];
    if (begin) begin[b] = nd->begin;
    if (end) end[b] = nd->end;
    if (left) left[b] = nd->left;
    if (right) right[b] = nd->right;
    if (radius) radius[b] = nd->radius;
    for (int a = 0; a < d; ++a) {
      if (center) center[(size_t)b * d + a] = nd->c[a];
      if (box_lo) box_lo[(size_t)b * d + a] = nd->lo[a];
      if (box_hi) box_hi[(size_t)b * d + a] = nd->hi[a];
    }
  }
}

/* ------------------------------------------------------------------------- */
/* Interaction sets: proj/src/tree.cpp:173-213, restated as a per-target
 * top-down walk (equivalent: a candidate reaches a node iff every ancestor
 * kept it), then a per-node ascending fill. */
int fko_tree_sets(fko_tree* t, double theta, long long* far_total, long long* near_total) {
  if (!(theta > 0.0 && theta < 1.0)) return -1;
  const int n = t->n, d = t->d, nodes = t->count;
  t->theta = theta;
  double* lim2 = (double*)malloc((size_t)nodes * sizeof(double));
  for (int b = 0; b < nodes; ++b) {
    const double limit = t->nodes[b].radius / theta;
    lim2[b] = limit * limit;
  }
  long long* fc = (long long*)calloc((size_t)nodes + 1, sizeof(long long));
  long long* nc = (long long*)calloc((size_t)nodes + 1, sizeof(long long));
  int* stack = (int*)malloc(((size_t)nodes + 1) * sizeof(int));
  /* pass 1: counts; pass 2: fill in ascending original index */
  uint32_t* posOf = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  for (int pos = 0; pos < n; ++pos) posOf[t->order[pos]] = (uint32_t)pos;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      free(t->far_off);
      free(t->near_off);
      free(t->far);
      free(t->near);
      t->far_off = (long long*)malloc(((size_t)nodes + 1) * sizeof(long long));
      t->near_off = (long long*)malloc(((size_t)nodes + 1) * sizeof(long long));
      long long a = 0, c = 0;
      for (int b = 0; b < nodes; ++b) {
        t->far_off[b] = a;
        t->near_off[b] = c;
        a += fc[b];
        c += nc[b];
        fc[b] = t->far_off[b];
        nc[b] = t->near_off[b];
      }
      t->far_off[nodes] = a;
      t->near_off[nodes] = c;
      t->far_total = a;
      t->near_total = c;
      t->far = (uint32_t*)malloc((size_t)(a > 0 ? a : 1) * sizeof(uint32_t));
      t->near = (uint32_t*)malloc((size_t)(c > 0 ? c : 1) * sizeof(uint32_t));
    }
    for (int orig = 0; orig < n; ++orig) {
      const double* pt = t->perm + (size_t)posOf[orig] * d;
      int sp = 0;
      stack[sp++] = 0;
      while (sp > 0) {
        const int b = stack[--sp];
        const fko_node* nd = &t->nodes[b];
        double dist2 = 0.0;
        for (int a = 0; a < d; ++a) {
          const double q = pt[a] - nd->c[a];
          dist2 += q * q;
        }
        if (dist2 > lim2[b]) {
          if (pass) t->far[fc[b]] = (uint32_t)orig;
          ++fc[b];
        } else if (nd->left < 0) {
          if (pass) t->near[nc[b]] = (uint32_t)orig;
          ++nc[b];
        } else {
          stack[sp++] = nd->right;
          stack[sp++] = nd->left;
        }
      }
    }
  }
  free(posOf);
  free(stack);
  free(fc);
  free(nc);
  free(lim2);
  *far_total = t->far_total;
  *near_total = t->near_total;
  return 0;
}

void fko_tree_set_arrays(const fko_tree* t, long long* far_off, uint32_t* far, long long* near_off, uint32_t* near) {
  const int nodes = t->count;
  if (far_off) memcpy(far_off, t->far_off, ((size_t)nodes + 1) * sizeof(long long));
  if (near_off) memcpy(near_off, t->near_off, ((size_t)nodes + 1) * sizeof(long long));
  if (far) memcpy(far, t->far, (size_t)t->far_total * sizeof(uint32_t));
  if (near) memcpy(near, t->near, (size_t)t->near_total * sizeof(uint32_t));
}

/* SURVEY Appendix A fingerprints (64-bit FNV-1a folds). */
void fko_fingerprints(int n, const uint32_t* order, int nodes, const long long* far_off, const uint32_t* far,
                      const long long* near_off, const uint32_t* near, const double* radius, const double* center,
                      int d, uint64_t out[3]) {
  const uint64_t P = 1099511628211ull;
  uint64_t ho = 1469598103934665603ull, hs = ho, hg = ho;
  for (int i = 0; i < n; ++i) {
    ho ^= order[i];
    ho *= P;
  }
  for (int b = 0; b < nodes; ++b) {
    for (long long i = far_off[b]; i < far_off[b + 1]; ++i) {
      hs ^= far[i] + (uint64_t)b * 0x9e3779b97f4a7c15ull;
      hs *= P;
    }
    for (long long i = near_off[b]; i < near_off[b + 1]; ++i) {
      hs ^= (uint64_t)near[i] * 31 + (uint64_t)b;
      hs *= P;
    }
    uint64_t bits;
    memcpy(&bits, &radius[b], 8);
    hg ^= bits;
    hg *= P;
    for (int a = 0; a < d; ++a) {
      memcpy(&bits, &center[(size_t)b * d + a], 8);
      hg ^= bits;
      hg *= P;
    }
  }
  out[0] = ho;
  out[1] = hs;
  out[2] = hg;
}

/* ------------------------------------------------------------------------- */
/* Kernels: proj/src/kernels.cpp:37-156 (double evaluators). prm = s2, a, is2, rho */
double fko_kernel(int id, const double* prm, double r) {
  const double s2 = prm[0], a = prm[1], is2 = prm[2], rho = prm[3];
  switch (id) {
    case 0: return exp(-r);
    case 1: return s2 * exp(-(r / rho));
    case 2: return s2 * (1.0 + a * r) * exp(-(a * r));
    case 3: return 1.0 / (1.0 + r * r * is2);
    case 4: return 1.0 / sqrt(1.0 + r * r * is2);
    case 5: return exp(-(r * r));
    case 6: return 1.0 / r;
    case 7: return 1.0 / (r * r);
    case 8: return 1.0 / (r * r * r);
    case 9: return exp(-r) / r;
    case 10: return r * exp(-r);
    case 11: return cos(r) / r;
    case 12: return exp(-(1.0 / r));
    case 13: return exp(-(1.0 / (r * r)));
  }
  return NAN;
}

/* Jets: proj/include/fkt/jet.hpp:110-190; c[m] = K^(m)(r)/m!, order p <= 32 */
#define JN 33
static void jmul(const double* a, const double* b, double* r, int n) {
  double t[JN] = {0};
  for (int i = 0; i <= n; ++i)
    for (int j = 0; j + i <= n; ++j) t[i + j] += a[i] * b[j];
  memcpy(r, t, (size_t)(n + 1) * sizeof(double));
}
static void jdiv(const double* a, const double* b, double* r, int n) {
  double t[JN];
  for (int i = 0; i <= n; ++i) {
    double acc = a[i];
    for (int j = 1; j <= i; ++j) acc -= b[j] * t[i - j];
    t[i] = acc / b[0];
  }
  memcpy(r, t, (size_t)(n + 1) * sizeof(double));
}
static void jexp(const double* f, double* g, int n) {
  double t[JN];
  t[0] = exp(f[0]);
  for (int m = 1; m <= n; ++m) {
    double acc = 0.0;
    for (int k = 1; k <= m; ++k) acc += k * f[k] * t[m - k];
    t[m] = acc / m;
  }
  memcpy(g, t, (size_t)(n + 1) * sizeof(double));
}
static void jsqrt(const double* f, double* g, int n) {
  double t[JN];
  t[0] = sqrt(f[0]);
  for (int m = 1; m <= n; ++m) {
    double acc = f[m];
    for (int k = 1; k < m; ++k) acc -= t[k] * t[m - k];
    t[m] = acc / (2.0 * t[0]);
  }
  memcpy(g, t, (size_t)(n + 1) * sizeof(double));
}
static void jcos(const double* f, double* c, int n) {
  double s[JN], cc[JN];
  s[0] = sin(f[0]);
  cc[0] = cos(f[0]);
  for (int m = 1; m <= n; ++m) {
    double sa = 0.0, ca = 0.0;
    for (int k = 1; k <= m; ++k) {
      const double kf = k * f[k];
      sa += kf * cc[m - k];
      ca -= kf * s[m - k];
    }
    s[m] = sa / m;
    cc[m] = ca / m;
  }
  memcpy(c, cc, (size_t)(n + 1) * sizeof(double));
}
static void jscale(double* a, double s, int n) {
  for (int i = 0; i <= n; ++i) a[i] *= s;
}
static void jconst(double* a, double v, int n) {
  memset(a, 0, (size_t)(n + 1) * sizeof(double));
  a[0] = v;
}

void fko_kernel_jet(int id, const double* prm, double r, int n, double* out) {
  const double s2 = prm[0], a = prm[1], is2 = prm[2], rho = prm[3];
  double v[JN] = {0}, t1[JN], t2[JN], one[JN];
  v[0] = r;
  if (n >= 1) v[1] = 1.0;
  jconst(one, 1.0, n);
  switch (id) {
    case 0: /* exp(-r) */
      memcpy(t1, v, sizeof(t1));
      jscale(t1, -1.0, n);
      jexp(t1, out, n);
      return;
    case 1: /* s2 * exp(-(r / rho)) ; Jet / double = * (1/rho) */
      memcpy(t1, v, sizeof(t1));
      jscale(t1, 1.0 / rho, n);
      jscale(t1, -1.0, n);
      jexp(t1, out, n);
      jscale(out, s2, n);
      return;
    case 2: /* s2 * (1 + a r) * exp(-(a r)) */
      memcpy(t1, v, sizeof(t1));
      jscale(t1, a, n);
      memcpy(t2, t1, sizeof(t2));
      t1[0] += 1.0;
      jscale(t1, s2, n);
      jscale(t2, -1.0, n);
      jexp(t2, t2, n);
      jmul(t1, t2, out, n);
      return;
    case 3: /* 1 / (1 + r r is2) */
      jmul(v, v, t1, n);
      jscale(t1, is2, n);
      t1[0] += 1.0;
      jdiv(one, t1, out, n);
      return;
    case 4:
      jmul(v, v, t1, n);
      jscale(t1, is2, n);
      t1[0] += 1.0;
      jsqrt(t1, t1, n);
      jdiv(one, t1, out, n);
      return;
    case 5:
      jmul(v, v, t1, n);
      jscale(t1, -1.0, n);
      jexp(t1, out, n);
      return;
    case 6:
      jdiv(one, v, out, n);
      return;
    case 7:
      jmul(v, v, t1, n);
      jdiv(one, t1, out, n);
      return;
    case 8:
      jmul(v, v, t1, n);
      jmul(t1, v, t1, n);
      jdiv(one, t1, out, n);
      return;
    case 9:
      memcpy(t1, v, sizeof(t1));
      jscale(t1, -1.0, n);
      jexp(t1, t1, n);
      jdiv(t1, v, out, n);
      return;
    case 10:
      memcpy(t1, v, sizeof(t1));
      jscale(t1, -1.0, n);
      jexp(t1, t1, n);
      jmul(v, t1, out, n);
      return;
    case 11:
      jcos(v, t1, n);
      jdiv(t1, v, out, n);
      return;
    case 12:
      jdiv(one, v, t1, n);
      jscale(t1, -1.0, n);
      jexp(t1, out, n);
      return;
    case 13:
      jmul(v, v, t1, n);
      jdiv(one, t1, t1, n);
      jscale(t1, -1.0, n);
      jexp(t1, out, n);
      return;
  }
}

/* ------------------------------------------------------------------------- */
/* Harmonics: proj/src/harmonics.cpp:160-246 (values scaled by the chain norm) */
static void harmonics(int d, int p, const double* point, const fko_tables* T, double* values, double* g, double* cA,
                      double* cB) {
  double norm2 = 0.0, v[64];
  for (int a = 0; a < d; ++a) norm2 += point[a] * point[a];
  const double inv = 1.0 / sqrt(norm2);
  for (int a = 0; a < d; ++a) v[a] = point[a] * inv;
  const double cx = v[d - 2], cy = v[d - 1];
  cA[0] = 1.0;
  cB[0] = 0.0;
  for (int m = 1; m <= p; ++m) {
    cA[m] = cA[m - 1] * cx - cB[m - 1] * cy;
    cB[m] = cB[m - 1] * cx + cA[m - 1] * cy;
  }
  if (d == 2) {
    for (int h = 0; h < T->H; ++h) {
      const int k = T->hdeg[h];
      values[h] = T->chain_norm[h] * (T->chain_phase[h] >= 0 ? cA[k] : cB[k]);
    }
    return;
  }
  double tail[64], acc = 0.0;
  for (int i = d - 1; i >= 0; --i) {
    acc += v[i] * v[i];
    tail[i] = acc;
  }
  const int W = p + 1;
  for (int level = 1; level <= d - 2; ++level) {
    const double x = v[level - 1], t2 = tail[level - 1];
    for (int m = 0; m <= p; ++m) {
      const double lambda = 0.5 * (d - 1 - level) + m;
      double* row = g + ((size_t)level * W + m) * W;
      row[0] = 1.0;
      if (p - m >= 1) row[1] = 2.0 * lambda * x;
      for (int nn = 2; nn <= p - m; ++nn)
        row[nn] = (2.0 * x * (nn + lambda - 1.0) * row[nn - 1] - t2 * (nn + 2.0 * lambda - 2.0) * row[nn - 2]) / nn;
    }
  }
  for (int h = 0; h < T->H; ++h) {
    const int* cm = T->chain_m + (size_t)h * (d - 1);
    double prod = T->chain_norm[h];
    for (int level = 1; level <= d - 2; ++level) {
      const int mi = cm[level], nn = cm[level - 1] - cm[level];
      prod *= g[((size_t)level * W + mi) * W + nn];
    }
    const int last = cm[d - 2];
    prod *= T->chain_phase[h] >= 0 ? cA[last] : cB[last];
    values[h] = prod;
  }
}

static double laurent_eval(const int* pw, const double* c, int lo, int hi, double r) {
  double acc = 0.0;
  for (int i = lo; i < hi; ++i) acc += c[i] * pow(r, pw[i]);
  return acc;
}

/* ------------------------------------------------------------------------- */
/* Multiply: proj/src/transform.cpp:127-204 (streaming operators rebuilt per
 * node: expansion.cpp:12-44 radial coefficients, :263-312 s2m, :314-355 m2t,
 * near field transform.cpp:163-181). Per-thread z buffers summed in thread
 * order (transform.cpp:194-203). */
int fko_multiply(const fko_tree* t, int kid, const double* prm, double diag, const fko_tables* T, const double* y,
                 double* z, int threads) {
  const int n = t->n, d = t->d, p = T->p, H = T->H, nodes = t->count;
  if (!t->far_off || p >= JN - 1 || d > 64) return -1;
  int slots[JN], coff[JN + 1], hoff[JN + 1], fstart[JN];
  int P = 0, f = 0;
  {
    int h = 0;
    for (int k = 0; k <= p; ++k) {
      hoff[k] = h;
      while (h < H && T->hdeg[h] == k) ++h;
      slots[k] = T->compressed ? T->ranks[k] : (p - k) / 2 + 1;
      coff[k] = P;
      P += (h - hoff[k]) * slots[k];
      fstart[k] = f;
      f += T->compressed ? T->ranks[k] : 0;
    }
    hoff[p + 1] = h;
    coff[p + 1] = P;
  }
  uint32_t* posOf = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  for (int pos = 0; pos < n; ++pos) posOf[t->order[pos]] = (uint32_t)pos;
#ifdef _OPENMP
  const int nth = threads > 0 ? threads : omp_get_max_threads();
#else
  const int nth = 1;
  (void)threads;
#endif
  double* zbuf = (double*)calloc((size_t)nth * n, sizeof(double));
#pragma omp parallel num_threads(nth)
  {
#ifdef _OPENMP
    const int tid = omp_get_thread_num();
#else
    const int tid = 0;
#endif
    double* zt = zbuf + (size_t)tid * n;
    const int W = p + 1;
    double* g = (double*)malloc((size_t)(d > 2 ? d - 1 : 1) * W * W * sizeof(double));
    double* Y = (double*)malloc((size_t)(H > 0 ? H : 1) * sizeof(double));
    double* mom = (double*)malloc((size_t)(P > 0 ? P : 1) * sizeof(double));
    double cA[JN], cB[JN], cj[JN], dk[JN], rel[64];
#pragma omp for schedule(dynamic, 1)
    for (int b = 0; b < nodes; ++b) {
      const fko_node* nd = &t->nodes[b];
      const long long f0 = t->far_off[b], f1 = t->far_off[b + 1];
      if (f1 > f0) {
        memset(mom, 0, (size_t)P * sizeof(double));
        for (uint32_t pos = nd->begin; pos < nd->end; ++pos) { /* moments = s2m * ySub */
          const double w = y[t->order[pos]];
          double r2 = 0.0;
          for (int a = 0; a < d; ++a) {
            rel[a] = t->perm[(size_t)pos * d + a] - nd->c[a];
            r2 += rel[a] * rel[a];
          }
          const double r = sqrt(r2);
          if (r == 0.0) { /* collocated source: degree-0 rows only (expansion.cpp:273-289) */
            const double y0 = 1.0 / sqrt(T->zk[0]);
            if (T->compressed) {
              for (int i = 0; i < slots[0]; ++i) {
                const int fi = fstart[0] + i;
                double c0 = 0.0;
                for (int q = T->src_off[fi]; q < T->src_off[fi + 1]; ++q)
                  if (T->src_pow[q] == 0) c0 = T->src_c[q];
                mom[coff[0] + i] += y0 * c0 * w;
              }
            } else {
              mom[coff[0]] += y0 * w;
            }
            continue;
          }
          harmonics(d, p, rel, T, Y, g, cA, cB);
          for (int k = 0; k <= p; ++k)
            for (int h = hoff[k]; h < hoff[k + 1]; ++h)
              for (int s = 0; s < slots[k]; ++s) {
                double rv;
                if (T->compressed) {
                  const int fi = fstart[k] + s;
                  rv = laurent_eval(T->src_pow, T->src_c, T->src_off[fi], T->src_off[fi + 1], r);
                } else {
                  rv = pow(r, k + 2 * s);
                }
                mom[coff[k] + (h - hoff[k]) * slots[k] + s] += Y[h] * rv * w;
              }
        }
        for (long long q = f0; q < f1; ++q) { /* z[far] += m2t * moments */
          const uint32_t tgt = t->far[q];
          const double* xt = t->perm + (size_t)posOf[tgt] * d; /* same values as the original cloud */
          double r2 = 0.0;
          for (int a = 0; a < d; ++a) {
            rel[a] = xt[a] - nd->c[a];
            r2 += rel[a] * rel[a];
          }
          const double r = sqrt(r2);
          harmonics(d, p, rel, T, Y, g, cA, cB);
          double acc = 0.0;
          if (T->compressed) {
            const double kv = fko_kernel(kid, prm, r);
            for (int k = 0; k <= p; ++k)
              for (int h = hoff[k]; h < hoff[k + 1]; ++h)
                for (int s = 0; s < slots[k]; ++s) {
                  const int fi = fstart[k] + s;
                  const double fr = laurent_eval(T->tgt_pow, T->tgt_c, T->tgt_off[fi], T->tgt_off[fi + 1], r);
                  acc += Y[h] * T->zk[k] * kv * fr * mom[coff[k] + (h - hoff[k]) * slots[k] + s];
                }
          } else {
            fko_kernel_jet(kid, prm, r, p, cj);
            double rm = 1.0, fact = 1.0;
            for (int m = 0; m <= p; ++m) {
              if (m > 0) fact *= m;
              dk[m] = cj[m] * fact * rm;
              rm *= r;
            }
            for (int k = 0; k <= p; ++k)
              for (int s = 0; s < slots[k]; ++s) {
                const int j = k + 2 * s;
                double wkj = 0.0;
                for (int m = 1; m <= j; ++m) wkj += dk[m] * T->tbar[((size_t)k * W + j) * W + m];
                wkj *= pow(r, -j);
                if (k == 0 && j == 0) wkj += fko_kernel(kid, prm, r);
                for (int h = hoff[k]; h < hoff[k + 1]; ++h)
                  acc += Y[h] * T->zk[k] * wkj * mom[coff[k] + (h - hoff[k]) * slots[k] + s];
              }
          }
          zt[tgt] += acc;
        }
      }
      if (nd->left < 0) { /* near field, exact dense block */
        for (long long q = t->near_off[b]; q < t->near_off[b + 1]; ++q) {
          const uint32_t tgt = t->near[q];
          const double* tp = t->perm + (size_t)posOf[tgt] * d;
          double acc = 0.0;
          for (uint32_t pos = nd->begin; pos < nd->end; ++pos) {
            const double* sp = t->perm + (size_t)pos * d;
            double dist2 = 0.0;
            for (int a = 0; a < d; ++a) {
              const double u = tp[a] - sp[a];
              dist2 += u * u;
            }
            const double r = sqrt(dist2);
            acc += (r == 0.0 ? diag : fko_kernel(kid, prm, r)) * y[t->order[pos]];
          }
          zt[tgt] += acc;
        }
      }
    }
    free(g);
    free(Y);
    free(mom);
  }
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int w = 0; w < nth; ++w) s += zbuf[(size_t)w * n + i];
    z[i] = s;
  }
  free(zbuf);
  free(posOf);
  return 0;
}

/* Dense rows: proj/src/transform.cpp:210-237 per row. */
int fko_dense_rows(int n, int d, const double* x, int kid, const double* prm, double diag, const double* y, int m,
                   const int64_t* rows, double* z, int threads) {
#ifdef _OPENMP
  const int nth = threads > 0 ? threads : omp_get_max_threads();
#else
  (void)threads;
#endif
#pragma omp parallel for num_threads(nth) schedule(dynamic, 4)
  for (int q = 0; q < m; ++q) {
    const double* pi = x + (size_t)rows[q] * d;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const double* pj = x + (size_t)j * d;
      double dist2 = 0.0;
      for (int a = 0; a < d; ++a) {
        const double u = pi[a] - pj[a];
        dist2 += u * u;
      }
      const double r = sqrt(dist2);
      acc += (r == 0.0 ? diag : fko_kernel(kid, prm, r)) * y[j];
    }
    z[q] = acc;
  }
  return 0;
}
