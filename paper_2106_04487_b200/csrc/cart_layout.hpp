// Layout of the Cartesian (q-form) M2T coefficients, shared by the host table
// builder (moments.cpp) and the device kernel (far.cu m2t_cart).
#ifndef FKTB_CART_LAYOUT_HPP
#define FKTB_CART_LAYOUT_HPP

#include "fkt_device_types.h"

namespace fktb {

// The far field of a node is the degree-p Taylor polynomial in the source
// offset x' of K(|x - x'|) = F(q + delta), q = |x|^2, delta = -2 x.x' + |x'|^2:
//   z_t = sum_n F^(n)(q)/n! Q_n(x),
//   Q_n(x) = sum_{i <= min(n, p-n)} binom(n,i) (-2)^(n-i) sum_src y (x.x')^(n-i) |x'|^(2i),
// Q_n a polynomial in x with homogeneous parts of degree n - i, i.e. degrees
// [cart_block_lo(p, n), n]. Monomials in nv variables with total degree in [lo, hi]:
constexpr int cart_count(int nv, int lo, int hi) {
  int c = 0;
  for (int a = lo; a <= hi; ++a) {
    // binom(a + nv - 1, nv - 1)
    long long b = 1;
    for (int i = 1; i <= nv - 1; ++i) b = b * (a + i) / i;
    c += static_cast<int>(b);
  }
  return c;
}
constexpr int cart_block_lo(int p, int n) { return 2 * n - p > 0 ? 2 * n - p : 0; }
// Kernels whose F^(n)(q) is a common factor (e^-q: the Gaussian) merge all
// blocks into one polynomial of degree <= p.
constexpr bool cart_merged(int kid) { return kid == FKTB_KERNEL_GAUSSIAN; }
constexpr int cart_block_offset(int kid, int d, int p, int n) {
  if (cart_merged(kid)) return 0;
  int c = 0;
  for (int m = 0; m < n; ++m) c += cart_count(d, cart_block_lo(p, m), m);
  return c;
}
constexpr int cart_total(int kid, int d, int p) {
  return cart_merged(kid) ? cart_count(d, 0, p) : cart_block_offset(kid, d, p, p + 1);
}

}  // namespace fktb

#endif
