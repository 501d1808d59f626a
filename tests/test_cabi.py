"""CPU: the C-ABI library loads, exports every symbol include/fkt_cuda.h
declares, and its host-side pieces (kernel registry, exact plan-time tables,
seeded inputs, error mapping) agree with the oracle / the reference. No
device compute here."""
import ctypes
import math
import os
import re
from fractions import Fraction as Q

import numpy as np
import pytest

from oracle import tables as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fkt_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fkt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(fkt):
    names = header_functions()
    assert len(names) >= 35
    lib = ctypes.CDLL(fkt._L.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table binds exactly those
    assert set(fkt._L.SIGNATURES) == set(names)


def test_cpp_api_library_exports(fkt):
    so = os.path.join(ROOT, "paper_2106_04487_b200", "lib", "libfkt.so")
    if not os.path.exists(so):
        pytest.skip("libfkt.so (C++ API) not built")
    out = os.popen(f"nm -DC {so}").read()
    for sym in ["fkt::FktPlan::FktPlan", "fkt::FktPlan::multiply", "fkt::PartitionTree::PartitionTree",
                "fkt::PartitionTree::computeInteractionSets", "fkt::makeKernel", "fkt::denseMultiply",
                "fkt::relativeError", "fkt::plan"]:
        assert sym in out, sym


def test_builtin_kernel_names(fkt):
    assert fkt.builtinKernelNames() == T.KERNELS


def test_make_kernel_validation(fkt):
    with pytest.raises(fkt.InvalidArgument):
        fkt.makeKernel("no-such-kernel")
    with pytest.raises(fkt.InvalidArgument):
        fkt.makeKernel("cauchy", {"rho": 1.0})  # unknown parameter (kernels.cpp:18-26)
    k = fkt.makeKernel("matern32", {"sigma": 2.0, "rho": 0.5})
    assert k.valueAtZero() == 4.0
    assert not k.hasDerivativeRecurrence()
    assert fkt.makeKernel("gaussian").hasDerivativeRecurrence()


def test_kernel_host_eval_and_diagonal(fkt, ref):
    # IsotropicKernel::operator() (kernels.hpp:49-58): r == 0 -> override, else convention
    k = fkt.makeKernel("inverse-r")
    assert k(0.0) == 0.0
    assert k(0.0, 5.0) == 5.0
    assert k(2.0) == 0.5
    for name in T.KERNELS:
        prm = {"sigma": 1.3, "rho": 0.4} if name.startswith("matern") else (
            {"sigma": 0.7} if name in ("cauchy", "rational-quadratic") else {})
        kk = fkt.makeKernel(name, prm)
        rs = np.array([0.05, 0.3, 1.0, 2.5])
        ours = kk(rs)
        refv = np.array([ref.kernel_jet(name, prm, r, 0)[0] for r in rs])
        np.testing.assert_allclose(ours, refv, rtol=1e-15)


@pytest.mark.parametrize("d,p", [(2, 6), (3, 4), (3, 8), (5, 4), (4, 6), (6, 3)])
def test_product_tbar_exact(fkt, d, p):
    tt = T.tbar_table(d, p)
    for (k, j, m), q in tt.items():
        v, s = fkt.tbar(d, p, k, j, m)
        assert Q(s) == q
        assert v == float(q)


def test_product_order_cap(fkt):
    with pytest.raises(fkt.OrderTooLargeError):
        fkt.tbar(3, 21, 0, 0, 1)


@pytest.mark.parametrize("name", ["gaussian", "inverse-r", "exponential", "r-exp", "exp-neg-inv-r2", "matern12"])
@pytest.mark.parametrize("d,p", [(2, 6), (3, 8), (5, 4), (4, 9)])
def test_product_compression_ranks(fkt, name, d, p):
    prm = {"sigma": 1.0, "rho": 0.3} if name == "matern12" else {}
    want = [r for r, _, _ in T.radial_compression(name, prm, d, p)]
    assert fkt.compressionRanks(fkt.makeKernel(name, prm), d, p) == want


def test_product_compression_requires_recurrence(fkt):
    with pytest.raises(fkt.NotRecurrenceKernelError):
        fkt.compressionRanks(fkt.makeKernel("matern32"), 3, 4)


def test_product_normalizers(fkt):
    for d in range(2, 8):
        for k in range(7):
            assert fkt.additionNormalizer(d, k) == pytest.approx(T.addition_normalizer(d, k), rel=1e-15)
    assert fkt.expansionSize(3, 6) == math.comb(9, 6) == 84


@pytest.mark.parametrize("cfg,n", [(1, 3000), (2, 3000), (3, 3000), (4, 3000), (5, 3000)])
def test_synthetic_inputs_bit_identical(fkt, ref, cfg, n):
    x, w = fkt.synthConfig(cfg, n)
    xr, wr = ref.gen_config(cfg, n)
    np.testing.assert_array_equal(x.view(np.uint64), xr.view(np.uint64))
    np.testing.assert_array_equal(np.asarray(w).view(np.uint64), np.asarray(wr).view(np.uint64))


@pytest.mark.parametrize("kind,d", [("cube", 3), ("sphere", 4), ("mixture", 5), ("sphere", 2)])
def test_synthetic_clouds_bit_identical(fkt, ref, kind, d):
    x, y = fkt.synthCloud(kind, 2000, d, 17)
    xr, yr = ref.gen_cloud(kind, 2000, d, 17)
    np.testing.assert_array_equal(x.view(np.uint64), xr.view(np.uint64))
    np.testing.assert_array_equal(y.view(np.uint64), yr.view(np.uint64))


def test_relative_error_host(fkt):
    assert fkt.relativeError([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert fkt.relativeError([1.01, 2.02], [1.0, 2.0]) == pytest.approx(0.01, rel=1e-12)
    with pytest.raises(fkt.ZeroReferenceError):
        fkt.relativeError([1.0, 2.0], [0.0, 0.0])
    with pytest.raises(fkt.DimensionMismatchError):
        fkt.relativeError([1.0], [1.0, 2.0])


def test_no_cpu_fallback(fkt):
    """Without a device the GPU path fails loudly (there is no CPU fallback)."""
    from conftest import has_gpu

    if has_gpu():
        pytest.skip("a GPU is present")
    x, w = fkt.synthConfig(1, 1000)
    with pytest.raises(fkt.CudaError):
        fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("cauchy"))
    with pytest.raises(fkt.CudaError):
        fkt.denseMultiply(fkt.PointCloud.from_array(x), fkt.makeKernel("cauchy"), w)
