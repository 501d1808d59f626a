"""The Cartesian (q-form) far field behind csrc/far.cu m2t_cart, restated in
NumPy and pinned to the unmodified reference FKT on the CPU (oracle/_ref):

    K(|x - x'|) = F(q + delta),  q = |x|^2,  delta = -2 x.x' + |x'|^2,
    z_t = sum_{n<=p} F^(n)(q)/n! sum_{i<=min(n,p-n)} C(n,i) (-2)^(n-i)
          sum_{|beta|=n-i} ((n-i)!/beta!) x^beta nu_{i,beta},
    nu_{i,beta} = sum_{|gamma|=i} (i!/gamma!) mu_{beta+2 gamma},  mu_a = sum_src y x'^a,

i.e. the degree-p Taylor polynomial in the source offset, which is what the
reference's Gegenbauer / harmonic expansion (expansion.cpp:12-55, 263-355)
evaluates. The near field is summed densely over the reference's own near
sets, the far field by the formula over its far sets; the total must equal the
reference FKT to rounding (far tighter than the 1e-10 gate), for the kernels
with a q-derivative form in the CUDA kernel (Matern-1/2 and -3/2, exponential,
Gaussian, Cauchy)."""
import itertools
import math

import numpy as np
import pytest


def _monomials(d, p):
    return [a for a in itertools.product(range(p + 1), repeat=d) if sum(a) <= p]


def _multinomial(a):
    r = math.factorial(sum(a))
    for v in a:
        r //= math.factorial(v)
    return r


def _phi(kernel, prm, q, p):
    """F^(n)(q)/n!, n = 0..p (the per-pair factors of m2t_cart)."""
    out = np.zeros((p + 1, len(q)))
    if kernel == "gaussian":
        for n in range(p + 1):
            out[n] = (-1.0) ** n * np.exp(-q) / math.factorial(n)
    elif kernel == "cauchy":
        is2 = 1.0 / prm["sigma"] ** 2
        F = 1.0 / (1.0 + q * is2)
        for n in range(p + 1):
            out[n] = (-is2) ** n * F ** (n + 1)
    elif kernel in ("exponential", "matern12"):  # e^(-a r): h_(n+1) = (h_(n-1) + (2n - 1) h_n) / u^2
        a = 1.0 if kernel == "exponential" else 1.0 / prm["rho"]
        s2 = 1.0 if kernel == "exponential" else prm["sigma"] ** 2
        u = a * np.sqrt(q)
        h = [np.exp(-u), np.exp(-u) / u]
        for n in range(1, p):
            h.append((h[n - 1] + (2 * n - 1) * h[n]) / u ** 2)
        for n in range(p + 1):
            out[n] = s2 * (a * a / 2) ** n * (-1.0) ** n * h[n] / math.factorial(n)
    else:  # matern32: h_(n+1) = (h_(n-1) + (2n - 3) h_n) / u^2
        a, s2 = math.sqrt(3.0) / prm["rho"], prm["sigma"] ** 2
        u = a * np.sqrt(q)
        h = [(1 + u) * np.exp(-u), np.exp(-u), np.exp(-u) / u]
        for n in range(2, p):
            h.append((h[n - 1] + (2 * n - 3) * h[n]) / u ** 2)
        for n in range(p + 1):
            out[n] = s2 * (a * a / 2) ** n * (-1.0) ** n * h[n] / math.factorial(n)
    return out


def _kernel(kernel, prm, r):
    if kernel == "gaussian":
        return np.exp(-r * r)
    if kernel == "cauchy":
        return 1.0 / (1.0 + r * r / prm["sigma"] ** 2)
    if kernel == "exponential":
        return np.exp(-r)
    if kernel == "matern12":
        return prm["sigma"] ** 2 * np.exp(-r / prm["rho"])
    a = math.sqrt(3.0) / prm["rho"]
    return prm["sigma"] ** 2 * (1 + a * r) * np.exp(-a * r)


@pytest.mark.parametrize("kernel,prm,d,p", [
    ("matern32", {"sigma": 1.0, "rho": 0.3}, 3, 6),
    ("gaussian", {}, 5, 4),
    ("gaussian", {}, 3, 6),
    ("cauchy", {"sigma": 1.0}, 3, 4),
    ("exponential", {}, 3, 4),
    ("matern12", {"sigma": 1.2, "rho": 0.4}, 3, 6),
])
def test_q_form_equals_reference_fkt(kernel, prm, d, p):
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(1)
    n = 900
    x = rng.random((n, d))
    w = rng.standard_normal(n)
    rp = ref.RefPlan(x, kernel, prm or None, p=p, theta=0.5, leaf=40)
    zr = rp.multiply(w)
    t = rp.tree()
    assert rp.far_total > 1000
    mons = _monomials(d, p)
    midx = {a: i for i, a in enumerate(mons)}
    by_deg = {k: [m for m in mons if sum(m) == k] for k in range(p + 1)}
    z = np.zeros(n)
    order = t["order"]
    for b in range(len(t["begin"])):
        src = order[t["begin"][b]:t["end"][b]]
        n0, n1 = t["nearOff"][b], t["nearOff"][b + 1]
        if n1 > n0:
            tg = t["near"][n0:n1]
            r = np.linalg.norm(x[tg][:, None, :] - x[src][None, :, :], axis=2)
            np.add.at(z, tg, _kernel(kernel, prm, r) @ w[src])
        f0, f1 = t["farOff"][b], t["farOff"][b + 1]
        if f1 == f0:
            continue
        c = t["center"][b]
        xs = x[src] - c
        mu = np.array([np.sum(w[src] * np.prod(xs ** np.array(a), axis=1)) for a in mons])
        tg = t["far"][f0:f1]
        xt = x[tg] - c
        phi = _phi(kernel, prm, np.sum(xt * xt, axis=1), p)
        acc = np.zeros(len(tg))
        for nn in range(p + 1):
            Q = np.zeros(len(tg))
            for i in range(min(nn, p - nn) + 1):
                a = nn - i
                for beta in by_deg[a]:
                    nu = sum(_multinomial(g) * mu[midx[tuple(bb + 2 * gg for bb, gg in zip(beta, g))]] for g in by_deg[i])
                    Q += math.comb(nn, i) * (-2.0) ** a * _multinomial(beta) * nu * np.prod(xt ** np.array(beta), axis=1)
            acc += phi[nn] * Q
        np.add.at(z, tg, acc)
    assert np.linalg.norm(z - zr) / np.linalg.norm(zr) <= 1e-13
