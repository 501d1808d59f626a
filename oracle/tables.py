"""TEST INFRASTRUCTURE ONLY — exact-rational restatement of the reference's
plan-time tables (checker for the product's host tables and input to the C
restatement fkt_oracle.c). Python's fractions.Fraction is the exact
arithmetic (the reference uses Boost.Multiprecision cpp_rational,
proj/include/fkt/exact.hpp:14-15).

Restated functions (reference file:line):
  bell(n, m)               proj/src/coefficients.cpp:12-17
  cosine_power(d, i)       proj/src/coefficients.cpp:19-43
  tbar_table(d, p)         proj/src/coefficients.cpp:52-95
  harmonic_count(d, k)     proj/src/harmonics.cpp:55-60
  chains(d, k)             proj/src/harmonics.cpp:62-103
  chain_norm(d, chain)     proj/src/harmonics.cpp:118-158 (with gegenbauerNormSq :24-29)
  addition_normalizer(d,k) proj/src/harmonics.cpp:114-116
  recurrence(kernel, prm)  proj/src/kernels.cpp:37-156 (q with K' = q K)
  radial_compression(...)  proj/src/expansion.cpp:116-243
"""
from __future__ import annotations

import math
from fractions import Fraction as Q
from typing import Dict, List, Optional, Tuple

KERNELS = ["exponential", "matern12", "matern32", "cauchy", "rational-quadratic", "gaussian", "inverse-r",
           "inverse-r2", "inverse-r3", "exp-over-r", "r-exp", "cos-over-r", "exp-neg-inv-r", "exp-neg-inv-r2"]


def binom(n: int, k: int) -> int:
    if k < 0 or n < 0 or k > n:
        return 0
    return math.comb(n, k)


def double_factorial(n: int) -> int:
    f = 1
    while n >= 2:
        f *= n
        n -= 2
    return f


def bell(n: int, m: int) -> Q:
    r = Q(double_factorial(2 * n - 2 * m - 1) * binom(2 * n - m - 1, m - 1), 2 ** n)
    return -r if (n + m) % 2 else r


def rising(a: Q, n: int) -> Q:
    p = Q(1)
    for i in range(n):
        p *= a + i
    return p


def cosine_power(d: int, i: int) -> List[Q]:
    out = [Q(0)] * (i + 1)
    for k in range(i % 2, i + 1, 2):
        lo, hi = (i - k) // 2, (i + k) // 2
        if d == 2:
            num = math.factorial(i) * (k if k else 1)
            out[k] = Q(num, 2 ** i * math.factorial(lo) * math.factorial(hi))
        else:
            alpha = Q(d - 2, 2)
            out[k] = Q(math.factorial(i)) * (alpha + k) / (Q(2 ** i * math.factorial(lo)) * rising(alpha, hi + 1))
    return out


def tbar_table(d: int, p: int) -> Dict[Tuple[int, int, int], Q]:
    """{(k, j, m): T-bar_kjm} for k <= j <= p, j == k mod 2, 1 <= m <= j."""
    A = [cosine_power(d, i) for i in range(p + 1)]
    t = {}
    for k in range(p + 1):
        for j in range(k, p + 1, 2):
            for m in range(1, j + 1):
                acc = Q(0)
                for n in range(max((j + k + 1) // 2, m), j + 1):
                    i = 2 * n - j
                    if i < k:
                        continue
                    term = binom(n, i) * A[i][k] * Q(2 ** i, math.factorial(n))
                    if i % 2:
                        term = -term
                    acc += term * bell(n, m)
                t[(k, j, m)] = acc
    return t


# --- harmonics -------------------------------------------------------------------
def harmonic_count(d: int, k: int) -> int:
    return binom(k + d - 1, k) - binom(k + d - 3, k - 2)


def chains(d: int, k: int) -> List[List[int]]:
    if d == 2:
        return [[0]] if k == 0 else [[k], [-k]]
    out: List[List[int]] = []

    def rec(levels_left, top, prefix):
        if levels_left == 1:
            for m in range(top + 1):
                out.append(prefix + [m])
                if m > 0:
                    out.append(prefix + [-m])
            return
        for m in range(top + 1):
            rec(levels_left - 1, m, prefix + [m])

    rec(d - 2, k, [])
    return out


def _gegenbauer_norm_sq(n: int, lam: float) -> float:
    log_num = math.log(math.pi) + (1.0 - 2.0 * lam) * math.log(2.0) + math.lgamma(n + 2.0 * lam)
    log_den = math.lgamma(n + 1.0) + math.log(n + lam) + 2.0 * math.lgamma(lam)
    return math.exp(log_num - log_den)


def chain_norm(d: int, k: int, chain: List[int]) -> float:
    phase = 1 if chain[-1] > 0 else (-1 if chain[-1] < 0 else 0)
    if d == 2:
        return 1.0 / math.sqrt(2.0 * math.pi if phase == 0 else math.pi)
    m = [k] + [abs(c) for c in chain]
    norm = 1.0
    for level in range(1, d - 1):
        lam = 0.5 * (d - 1 - level) + m[level]
        norm /= _gegenbauer_norm_sq(m[level - 1] - m[level], lam)
    norm /= 2.0 * math.pi if phase == 0 else math.pi
    return math.sqrt(norm)


def gegenbauer_at_one(d: int, k: int) -> float:
    if d == 2:
        return 1.0 if k == 0 else 2.0 / k
    return float(binom(k + d - 3, k))


def addition_normalizer(d: int, k: int) -> float:
    surface = 2.0 * math.pi ** (0.5 * d) / math.gamma(0.5 * d)
    return surface * gegenbauer_at_one(d, k) / harmonic_count(d, k)


# --- kernels / compression ---------------------------------------------------------
Laurent = Dict[int, Q]  # power -> coefficient


def _ladd(a: Laurent, power: int, c: Q) -> None:
    if c == 0:
        return
    v = a.get(power, Q(0)) + c
    if v == 0:
        a.pop(power, None)
    else:
        a[power] = v


def recurrence(kernel: str, params: Optional[Dict[str, float]] = None) -> Optional[Laurent]:
    params = params or {}
    if kernel == "exponential":
        return {0: Q(-1)}
    if kernel == "matern12":
        return {0: -1 / Q(params.get("rho", 1.0))}
    if kernel == "gaussian":
        return {1: Q(-2)}
    if kernel == "inverse-r":
        return {-1: Q(-1)}
    if kernel == "inverse-r2":
        return {-1: Q(-2)}
    if kernel == "inverse-r3":
        return {-1: Q(-3)}
    if kernel == "exp-over-r":
        return {0: Q(-1), -1: Q(-1)}
    if kernel == "r-exp":
        return {-1: Q(1), 0: Q(-1)}
    if kernel == "exp-neg-inv-r":
        return {-2: Q(1)}
    if kernel == "exp-neg-inv-r2":
        return {-3: Q(2)}
    return None  # matern32, cauchy, rational-quadratic, cos-over-r


def _lmul(a: Laurent, b: Laurent) -> Laurent:
    r: Laurent = {}
    for p1, c1 in a.items():
        for p2, c2 in b.items():
            _ladd(r, p1 + p2, c1 * c2)
    return r


def _lderiv(a: Laurent) -> Laurent:
    r: Laurent = {}
    for p, c in a.items():
        if p != 0:
            _ladd(r, p - 1, c * p)
    return r


def _rank_revealing_qr(mat: List[List[Q]]):
    rows, cols = len(mat), len(mat[0]) if mat else 0
    work = [[mat[i][j] for i in range(rows)] for j in range(cols)]
    used = [False] * cols
    qcols, rrows = [], []
    for _ in range(min(rows, cols)):
        pivot, best = -1, Q(0)
        for j in range(cols):
            if used[j]:
                continue
            norm = sum((x * x for x in work[j]), Q(0))
            if pivot < 0 or norm > best:
                pivot, best = j, norm
        if pivot < 0 or best == 0:
            break
        used[pivot] = True
        q = list(work[pivot])
        rrow = [Q(0)] * cols
        rrow[pivot] = Q(1)
        for j in range(cols):
            if used[j]:
                continue
            proj = sum((q[i] * work[j][i] for i in range(rows)), Q(0)) / best
            if proj == 0:
                continue
            rrow[j] = proj
            work[j] = [work[j][i] - proj * q[i] for i in range(rows)]
        qcols.append(q)
        rrows.append(rrow)
    return qcols, rrows


def radial_compression(kernel: str, params, d: int, p: int):
    """[(rank, [target Laurent], [source Laurent]) per degree k] or None (no recurrence)."""
    q = recurrence(kernel, params)
    if q is None:
        return None
    t = tbar_table(d, p)
    lau = [{0: Q(1)}]
    for m in range(1, p + 1):
        nxt = _lderiv(lau[-1])
        for pw, c in _lmul(lau[-1], q).items():
            _ladd(nxt, pw, c)
        lau.append(nxt)
    out = []
    for k in range(p + 1):
        coeffs: Dict[int, Dict[int, Q]] = {}
        for j in range(k, p + 1, 2):
            for m in range(1, j + 1):
                tv = t[(k, j, m)]
                if tv == 0:
                    continue
                for pw, c in lau[m].items():
                    row = coeffs.setdefault(pw + m - j, {})
                    row[j] = row.get(j, Q(0)) + c * tv
            if k == 0 and j == 0:
                row = coeffs.setdefault(0, {})
                row[0] = row.get(0, Q(0)) + 1
        r_powers = sorted(coeffs)
        src_powers = list(range(k, p + 1, 2))
        mat = [[coeffs[rp].get(sp, Q(0)) for sp in src_powers] for rp in r_powers]
        qcols, rrows = _rank_revealing_qr(mat)
        tf = [{r_powers[i]: qc[i] for i in range(len(r_powers)) if qc[i] != 0} for qc in qcols]
        sf = [{src_powers[j]: rr[j] for j in range(len(src_powers)) if rr[j] != 0} for rr in rrows]
        out.append((len(qcols), tf, sf))
    return out
