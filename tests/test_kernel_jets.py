"""Host-side kernel jets and derivative recurrences of the C++ operator API
(IsotropicKernel::jetAt / evalJet / derivativeRecurrence, reference
kernels.hpp:61-68, kernels.cpp:37-156), through the C-ABI
(fkt_kernel_eval_jet, fkt_kernel_recurrence). No GPU needed."""
import ctypes as C
import math
from fractions import Fraction

import numpy as np
import pytest

KERNELS = [
    ("exponential", {}), ("matern12", {"sigma": 1.3, "rho": 0.7}), ("matern32", {"sigma": 0.9, "rho": 0.4}),
    ("cauchy", {"sigma": 0.8}), ("rational-quadratic", {"sigma": 1.1}), ("gaussian", {}), ("inverse-r", {}),
    ("inverse-r2", {}), ("inverse-r3", {}), ("exp-over-r", {}), ("r-exp", {}), ("cos-over-r", {}),
    ("exp-neg-inv-r", {}), ("exp-neg-inv-r2", {}),
]


def _params(fkt, prm):
    k, v, n = fkt._params(prm)
    return k, v, n


def jet_at(fkt, name, prm, r, order):
    k, v, n = _params(fkt, prm)
    arg = np.zeros(order + 1)
    arg[0] = r
    if order >= 1:
        arg[1] = 1.0
    out = np.zeros(order + 1)
    fkt._check(fkt.lib.fkt_kernel_eval_jet(name.encode(), k, v, n, r, order,
                                           arg.ctypes.data_as(C.POINTER(C.c_double)),
                                           out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def recurrence(fkt, name, prm):
    k, v, n = _params(fkt, prm)
    terms = C.c_int()
    powers = (C.c_int * 16)()
    buf = C.create_string_buffer(1 << 14)
    fkt._check(fkt.lib.fkt_kernel_recurrence(name.encode(), k, v, n, C.byref(terms), powers, 16, buf, len(buf)))
    texts = buf.raw.split(b"\0")[: terms.value]
    return {powers[i]: Fraction(texts[i].decode()) for i in range(terms.value)}


@pytest.mark.parametrize("name,prm", KERNELS)
def test_jet_value_and_slope(fkt, name, prm):
    for r in (0.3, 1.0, 2.7):
        c = jet_at(fkt, name, prm, r, 6)
        k0 = fkt.makeKernel(name, prm)
        assert abs(c[0] - k0(r)) <= 1e-14 * max(1.0, abs(c[0]))
        h = 1e-5 * r
        fd = (k0(r + h) - k0(r - h)) / (2 * h)
        assert abs(c[1] - fd) <= 1e-7 * max(1.0, abs(fd))
        # second derivative / 2 against a five-point difference
        fd2 = (-k0(r + 2 * h) + 16 * k0(r + h) - 30 * k0(r) + 16 * k0(r - h) - k0(r - 2 * h)) / (12 * h * h)
        assert abs(2 * c[2] - fd2) <= 1e-4 * max(1.0, abs(fd2))


def test_jet_exponential_closed_form(fkt):  # reference test_kernels.cpp:33-38
    c = jet_at(fkt, "exponential", {}, 1.0, 3)
    for m in range(4):
        assert abs(c[m] - math.exp(-1.0) * (-1) ** m / math.factorial(m)) <= 1e-15


@pytest.mark.parametrize("name,prm", KERNELS)
def test_recurrences_exact_and_consistent(fkt, name, prm):
    q = recurrence(fkt, name, prm)
    has = fkt.makeKernel(name, prm).hasDerivativeRecurrence()
    assert bool(q) == has
    if not q:
        return
    for r in (0.4, 1.3):
        c = jet_at(fkt, name, prm, r, 1)
        qr = sum(float(v) * r ** p for p, v in q.items())
        assert abs(c[1] - qr * c[0]) <= 1e-13 * max(1.0, abs(c[1]))


def test_recurrence_parameters_are_exact(fkt):
    q = recurrence(fkt, "matern12", {"sigma": 1.0, "rho": 0.7})
    assert q == {0: -1 / Fraction(0.7)}  # the exact dyadic rational of the double 0.7
    assert recurrence(fkt, "gaussian", {}) == {1: Fraction(-2)}
    assert recurrence(fkt, "exp-over-r", {}) == {-1: Fraction(-1), 0: Fraction(-1)}
