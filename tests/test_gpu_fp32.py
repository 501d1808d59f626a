"""FP32 fast near-field mode (north star: "plus an fp32 fast mode"): same
plan, same far field (FP64); the near-field pair kernel runs in FP32 with
leaf-centred coordinates and FP64 accumulation across leaves. Pinned against
the FP64 path: relative z error at the FP32 level, never a different
algorithm."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    ("matern32", {"sigma": 1.0, "rho": 0.1}, "cube", 3, 6),
    ("cauchy", {"sigma": 1.0}, "mixture", 2, 6),
    ("gaussian", {}, "mixture", 5, 4),
    ("inverse-r", {}, "sphere", 3, 6),
    ("exponential", {}, "cube", 3, 4),
]


@pytest.mark.parametrize("name,params,kind,d,p", CASES)
def test_fp32_near_close_to_fp64(fkt, name, params, kind, d, p):
    x, y = fkt.synthCloud(kind, 60000, d, 5)
    k = fkt.makeKernel(name, params)
    o64 = fkt.FktOptions(p=p, theta=0.5, leafCapacity=256)
    o32 = fkt.FktOptions(p=p, theta=0.5, leafCapacity=256, nearPrecision=32)
    z64 = fkt.plan(fkt.PointCloud.from_array(x), k, o64).multiply(y)
    z32 = fkt.plan(fkt.PointCloud.from_array(x), k, o32).multiply(y)
    err = fkt.relativeError(z32, z64)
    assert err < 2e-5, err
    assert err > 0.0  # it really ran the FP32 kernel


def test_fp32_multi_rhs(fkt):
    x, W = fkt.synthConfig(5, 40000)
    k = fkt.makeKernel("cauchy", {"sigma": 1.0})
    z64 = fkt.plan(fkt.PointCloud.from_array(x), k, fkt.FktOptions(p=6, leafCapacity=512)).multiply(W)
    z32 = fkt.plan(fkt.PointCloud.from_array(x), k, fkt.FktOptions(p=6, leafCapacity=512, nearPrecision=32)).multiply(W)
    for r in range(W.shape[1]):
        assert fkt.relativeError(z32[:, r], z64[:, r]) < 2e-5


def test_fp32_invalid_precision(fkt):
    x, y = fkt.synthCloud("cube", 100, 3, 1)
    with pytest.raises(fkt.InvalidArgument):
        fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("cauchy"), fkt.FktOptions(nearPrecision=16))
