"""Multi-RHS M2T on the FP64 tensor cores (csrc/far.cu m2t_mma):
nrhs % 8 == 0 and a basis of <= 64 coefficients take the DMMA GEMM path
(NT = 2 for nrhs % 16 == 0, else NT = 1 over 8-column groups). Every column is
checked against the unmodified reference FKT (oracle/_ref) at the 1e-10 gate,
and against the same plan's single-RHS multiply at 5e-12 (Matern-3/2 and
Gaussian plans run the Cartesian M2T there, a different evaluation of the same
polynomial: the two agree to 6e-14 for Matern-3/2; the compressed Gaussian's
harmonic form carries ~1e-12 of its own against the reference)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,prm,d,p,nrhs,comp", [
    ("cauchy", {"sigma": 1.0}, 2, 6, 16, None),            # cfg5 shape, NT = 2
    ("cauchy", {"sigma": 0.3}, 2, 6, 8, None),             # NT = 1
    ("matern32", {"sigma": 1.0, "rho": 0.2}, 2, 6, 24, None),  # 3 groups of 8
    ("gaussian", {}, 3, 4, 16, "on"),                       # compressed, PU = 35 (K padded to 36)
    ("inverse-r", {}, 3, 4, 32, "on"),                      # compressed singular kernel, 2 groups of 16
    ("cauchy", {"sigma": 1.0}, 3, 4, 8, "off"),
])
def test_mma_m2t_columns(fkt, ref, name, prm, d, p, nrhs, comp):
    rng = np.random.default_rng(21)
    n = 12000
    x = rng.random((n, d))
    W = rng.standard_normal((n, nrhs))
    mode = {None: fkt.CompressionMode.Auto, "on": fkt.CompressionMode.On, "off": fkt.CompressionMode.Off}[comp]
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                  fkt.FktOptions(p=p, theta=0.6, leafCapacity=128, compression=mode))
    Z = pl.multiply(W)
    rp = ref.RefPlan(x, name, prm, p=p, theta=0.6, leaf=128, compression=int(mode))
    for c in range(nrhs):
        col = np.ascontiguousarray(W[:, c])
        assert fkt.relativeError(Z[:, c], rp.multiply(col)) <= 1e-10, (c,)
        assert fkt.relativeError(Z[:, c], pl.multiply(col)) <= 5e-12, (c,)


@pytest.mark.parametrize("name,prm,d,p,nrhs,comp", [
    ("matern32", {"sigma": 1.0, "rho": 0.3}, 3, 6, 16, None),  # P2M RB = 16 (3 monomials / lane); M2T DFMA (P > 64)
    ("inverse-r", {}, 3, 8, 8, "on"),                           # P2M RB = 8 (6 monomials / lane)
    ("gaussian", {}, 5, 4, 8, "on"),                            # P2M RB = 8 (4 monomials / lane)
])
def test_rhs_blocked_p2m_columns(fkt, ref, name, prm, d, p, nrhs, comp):
    # RHS-blocked P2M (csrc/moments.cu p2m_multi) at the remaining moment
    # shapes: every column against the reference and the single-RHS path
    rng = np.random.default_rng(22)
    n = 10000
    x = rng.random((n, d))
    W = rng.standard_normal((n, nrhs))
    mode = {None: fkt.CompressionMode.Auto, "on": fkt.CompressionMode.On}[comp]
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                  fkt.FktOptions(p=p, theta=0.6, leafCapacity=256, compression=mode))
    Z = pl.multiply(W)
    rp = ref.RefPlan(x, name, prm, p=p, theta=0.6, leaf=256, compression=int(mode))
    for c in (0, nrhs // 2, nrhs - 1):
        col = np.ascontiguousarray(W[:, c])
        assert fkt.relativeError(Z[:, c], rp.multiply(col)) <= 1e-10, (c,)
        assert fkt.relativeError(Z[:, c], pl.multiply(col)) <= 5e-12, (c,)
