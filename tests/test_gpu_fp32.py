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


# --- pinned against the reference FKT (oracle/_ref) --------------------------
# FP32 near field: the pair kernel values carry FP32 rounding (~6e-8 relative
# each, leaf-centred coordinates), summed in FP32 per leaf block and in FP64
# across blocks. Stated tolerance against the reference FKT's z (FP64):
FP32_TOL = 5e-5
FP32_KERNELS = [("exponential", {}), ("matern12", {"sigma": 1.3, "rho": 0.7}), ("matern32", {"sigma": 0.9, "rho": 0.4}),
                ("cauchy", {"sigma": 0.8}), ("rational-quadratic", {"sigma": 1.1}), ("gaussian", {}),
                ("inverse-r", {}), ("inverse-r2", {})]


@pytest.mark.parametrize("name,prm", FP32_KERNELS)
@pytest.mark.parametrize("d", [2, 3, 5])
def test_fp32_vs_reference_fkt(fkt, ref, name, prm, d):
    x, y = fkt.synthCloud("cube", 20000, d, 11)
    opts = dict(p=4, theta=0.5, leafCapacity=256)
    z32 = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                   fkt.FktOptions(nearPrecision=32, **opts)).multiply(y)
    rp = ref.RefPlan(x, name, prm, p=4, theta=0.5, leaf=256)
    zr = rp.multiply(y)
    err = fkt.relativeError(z32, zr)
    assert 0.0 < err <= FP32_TOL, err


@pytest.mark.parametrize("cfg", [1, 2, 3, 5, 4])
def test_fp32_full_configs_vs_reference_rows(fkt, cfg):
    """The five BASELINE configurations at full size in FP32 mode, against the
    reference FKT's z on the golden rows (tests/golden, made by the unmodified
    reference); the FKT-vs-dense accuracy is unchanged at the FP32 level."""
    import json
    import os

    g = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    if not os.path.exists(os.path.join(g, f"cfg{cfg}_ref.json")):
        pytest.skip("golden fixture missing")
    meta = json.load(open(os.path.join(g, f"cfg{cfg}_ref.json")))
    gold = np.load(os.path.join(g, f"cfg{cfg}_ref.npz"))
    c = {1: ("cauchy", {"sigma": 1.0}, 20000, 4, 512, 0.5), 2: ("matern32", {"sigma": 1.0, "rho": 0.1}, 1000000, 6, 512, 0.5),
         3: ("gaussian", {}, 1000000, 4, 1024, 0.75), 4: ("inverse-r", {}, 4000000, 8, 512, 0.5),
         5: ("cauchy", {"sigma": 1.0}, 2000000, 6, 512, 0.75)}[cfg]
    x, w = fkt.synthConfig(cfg, c[2])
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(c[0], c[1]),
                  fkt.FktOptions(p=c[3], theta=c[5], leafCapacity=c[4], nearPrecision=32))
    z = pl.multiply(w)
    rows = gold["rows"]
    zr = z[rows] if z.ndim == 1 else z[rows, :]
    err = np.linalg.norm(zr - gold["z_rows"]) / np.linalg.norm(gold["z_rows"])
    assert 0.0 < err <= FP32_TOL, err
    zc = zr if zr.ndim == 1 else zr[:, 0]
    acc = np.linalg.norm(zc - gold["dense_rows"]) / np.linalg.norm(gold["dense_rows"])
    assert abs(acc - meta["fkt_vs_dense_rows"]) <= FP32_TOL + 1e-3 * meta["fkt_vs_dense_rows"]
