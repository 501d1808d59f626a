"""Cartesian (q-form) M2T of single-RHS multiplies (csrc/far.cu m2t_cart,
csrc/moments.cpp buildCartTable): the far field of a node as the
degree-p Taylor polynomial in the source offset, evaluated per pair as
sum_n F^(n)(q)/n! Q_n(x). Checked against the unmodified reference FKT
(expansion.cpp:12-55, 314-355 through oracle/_ref) at the 1e-10 gate, against
the harmonic M2T of the same plan (a two-column multiply takes it), and for
bitwise repeatability in deterministic mode. Kernels: Matern-1/2 and -3/2,
exponential, Gaussian, Cauchy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    ("matern32", {"sigma": 1.0, "rho": 0.1}, 3, 6, None),   # cfg2 shape
    ("matern32", {"sigma": 1.3, "rho": 0.4}, 3, 4, None),
    ("matern32", {"sigma": 0.7, "rho": 0.25}, 3, 8, None),
    ("matern32", {"sigma": 1.0, "rho": 0.2}, 3, 6, "off"),
    ("gaussian", {}, 5, 4, "on"),                           # cfg3 shape
    ("gaussian", {}, 3, 6, "on"),
    ("gaussian", {}, 3, 8, "off"),
    ("gaussian", {}, 3, 4, None),
    ("cauchy", {"sigma": 1.0}, 3, 4, None),                 # cfg1 shape
    ("cauchy", {"sigma": 0.3}, 3, 6, None),
    ("cauchy", {"sigma": 2.0}, 5, 4, None),
    ("exponential", {}, 3, 6, None),                        # compressed by default (same Taylor polynomial)
    ("exponential", {}, 3, 4, "off"),
    ("matern12", {"sigma": 1.2, "rho": 0.3}, 3, 8, None),
    ("matern12", {"sigma": 0.8, "rho": 0.5}, 5, 4, "off"),
]


def _mode(fkt, comp):
    return {None: fkt.CompressionMode.Auto, "on": fkt.CompressionMode.On, "off": fkt.CompressionMode.Off}[comp]


@pytest.mark.parametrize("name,prm,d,p,comp", CASES)
def test_cartesian_m2t_matches_reference_and_harmonic_path(fkt, ref, name, prm, d, p, comp):
    rng = np.random.default_rng(100 + 10 * d + p)
    n = 15000
    x = rng.random((n, d))
    y = rng.standard_normal(n)
    mode = _mode(fkt, comp)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                  fkt.FktOptions(p=p, theta=0.5, leafCapacity=128, compression=mode))
    assert pl.info()["m2t_cartesian"] == 1
    z = pl.multiply(y)                                     # Cartesian M2T
    Z2 = pl.multiply(np.stack([y, -2.0 * y], axis=1))      # harmonic M2T (nrhs = 2)
    rp = ref.RefPlan(x, name, prm, p=p, theta=0.5, leaf=128, compression=int(mode))
    zr = rp.multiply(y)
    assert rp.far_total > 0
    assert fkt.relativeError(z, zr) <= 1e-10
    # two evaluations of the same polynomial: 6e-14 apart for Matern-3/2; the
    # compressed Gaussian's harmonic form is ~1e-12 from the reference itself
    # (the Cartesian form 4e-13), so the bound between them is 5e-12
    assert fkt.relativeError(z, Z2[:, 0]) <= 5e-12
    assert fkt.relativeError(-2.0 * z, Z2[:, 1]) <= 5e-12
    assert fkt.relativeError(z, zr) <= 2.0 * fkt.relativeError(Z2[:, 0], zr) + 1e-13


def test_cartesian_m2t_not_used_for_other_kernels(fkt):
    rng = np.random.default_rng(5)
    x = rng.random((4000, 3))
    for name, prm, p in [("rational-quadratic", {"sigma": 1.0}, 4), ("inverse-r", {}, 8)]:
        pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm), fkt.FktOptions(p=p, leafCapacity=128))
        assert pl.info()["m2t_cartesian"] == 0
    # d = 2 keeps the harmonic form (28 coefficients against 50)
    pl = fkt.plan(fkt.PointCloud.from_array(rng.random((4000, 2))), fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.2}),
                  fkt.FktOptions(p=6, leafCapacity=128))
    assert pl.info()["m2t_cartesian"] == 0


def test_cartesian_m2t_deterministic_and_rebuild(fkt, ref):
    rng = np.random.default_rng(6)
    n = 20000
    x = rng.random((n, 3))
    y = rng.standard_normal(n)
    prm = {"sigma": 1.0, "rho": 0.15}
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("matern32", prm),
                  fkt.FktOptions(p=6, theta=0.5, leafCapacity=256, deterministic=True))
    z0 = pl.multiply(y)
    assert np.array_equal(z0, pl.multiply(y))
    x2 = rng.random((n, 3))
    pl.rebuild(fkt.PointCloud.from_array(x2))
    z2 = pl.multiply(y)
    zr = ref.RefPlan(x2, "matern32", prm, p=6, theta=0.5, leaf=256).multiply(y)
    assert fkt.relativeError(z2, zr) <= 1e-10
