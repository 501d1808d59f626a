// Source-to-multipole through monomial moments (product code).
//
// Every s2m row of the reference (proj/src/expansion.cpp:263-312) is a
// polynomial in the source offset x' = x - c of degree <= p:
//   Y_kh(x'/|x'|) |x'|^j = |x'|^(j-k) S_kh(x')       (S_kh: solid harmonic, degree k)
// and the compressed rows are combinations G_ki of those. So the node moments
// are a fixed linear map T of the monomial moments mu_a = sum y x'^a
// (|a| <= p), and monomial moments shift exactly between centers
// (multinomial binomial theorem). The GPU computes mu on the leaves from their
// sources (N source visits instead of N x depth), shifts them up the tree, and
// applies T per node. Same moments as the direct evaluation up to rounding.
#ifndef FKTB_MOMENTS_HPP
#define FKTB_MOMENTS_HPP

#include <vector>

#include "fkt_device_types.h"
#include "tables.hpp"

namespace fktb {

// Monomials x^a with |a| <= p in d variables, enumerated lexicographically by
// (a_0, a_1, ..., a_{d-1}) ascending with the total-degree bound: the order
// the device recursion (moments.cu) generates them in.
struct MonomialBasis {
  int d = 0, p = 0;
  std::vector<std::vector<int>> exps;
  int count() const { return static_cast<int>(exps.size()); }
  int index(const std::vector<int>& a) const;
  MonomialBasis(int d, int p);
};

struct MomentTables {
  int count = 0;                    // monomials
  std::vector<double> T;            // P (padded layout) x count, hscale folded
  // shift: mu_parent[a] += sum_e coef[e] * delta^mono[g[e]] * mu_child[b[e]],
  // entries of output a at [off[a], off[a+1]).
  std::vector<int> off, b, g;
  std::vector<double> coef;
};

// Coefficient layout as FktbFarParams (cOff/hOff/slotsU/slots); hscale per
// harmonic (Z_k nrm^2); factors for compressed plans (else empty).
MomentTables buildMomentTables(int d, int p, const HarmonicStructure& hs, const std::vector<RadialFactor>& factors,
                               bool compressed, const std::vector<double>& hscale);

// Cartesian M2T coefficients (far.cu m2t_cart): rows of the map from the
// monomial moments to the coefficients of the polynomials Q_n(x) (layout and
// formula in device_math.cuh), in the order the device Horner recursion reads
// them, with the kernel's constant factor of F^(n)(q)/n! folded in. Returns
// PCart x count (row-major); empty if the kernel has no Cartesian path.
std::vector<double> buildCartTable(int d, int p, const FktbKernelDesc& kernel, int& PCart);
bool cartSupported(int kid, int d, int p);

}  // namespace fktb

#endif
