"""GPU parity against the reference FKT (oracle/_ref = the unmodified
reference sources). Bit-exact tree and interaction sets; z within rel-L2
1e-10 in fp64 (BASELINE.json north star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10  # fp64 z vs the reference FKT (north_star)


def _tree_equal(gpu_tree, rt):
    assert gpu_tree.nodeCount() == len(rt["begin"])
    np.testing.assert_array_equal(gpu_tree.order(), rt["order"])
    np.testing.assert_array_equal(gpu_tree.begins, rt["begin"])
    np.testing.assert_array_equal(gpu_tree.ends, rt["end"])
    np.testing.assert_array_equal(gpu_tree.lefts, rt["left"])
    np.testing.assert_array_equal(gpu_tree.rights, rt["right"])
    # bit-exact geometry
    np.testing.assert_array_equal(gpu_tree.radii.view(np.uint64), rt["radius"].view(np.uint64))
    np.testing.assert_array_equal(gpu_tree.centers.view(np.uint64), rt["center"].view(np.uint64))
    np.testing.assert_array_equal(gpu_tree.boxLos.view(np.uint64), rt["boxLo"].view(np.uint64))
    np.testing.assert_array_equal(gpu_tree.boxHis.view(np.uint64), rt["boxHi"].view(np.uint64))
    np.testing.assert_array_equal(gpu_tree.points().view(np.uint64), rt["perm"].view(np.uint64))


def _sets_equal(gpu_tree, rt):
    fo, fi = gpu_tree.farCsr()
    no, ni = gpu_tree.nearCsr()
    np.testing.assert_array_equal(fo, rt["farOff"])
    np.testing.assert_array_equal(fi, rt["far"])
    np.testing.assert_array_equal(no, rt["nearOff"])
    np.testing.assert_array_equal(ni, rt["near"])


def test_cfg1_tree_sets_and_z(fkt, ref):
    x, w = fkt.synthConfig(1, 20000)
    xr, wr = ref.gen_config(1, 20000)
    np.testing.assert_array_equal(x, xr)
    np.testing.assert_array_equal(w, wr)
    k = fkt.makeKernel("cauchy", {"sigma": 1.0})
    opts = fkt.FktOptions(p=4, theta=0.5, leafCapacity=512)
    p = fkt.plan(fkt.PointCloud.from_array(x), k, opts)
    rp = ref.RefPlan(x, "cauchy", {"sigma": 1.0}, p=4, theta=0.5, leaf=512)
    rt = rp.tree()
    _tree_equal(p.tree(), rt)
    _sets_equal(p.tree(), rt)
    assert p.coefficientCount() == rp.coef == 35
    assert p.compressed() == rp.compressed
    z = p.multiply(w)
    zr = rp.multiply(w)
    err = fkt.relativeError(z, zr)
    assert err <= TOL, err
    # and the FKT itself is a good MVM (3.42e-4 vs dense)
    zd = fkt.denseMultiply(fkt.PointCloud.from_array(x), k, w)
    zdr = ref.dense(x, "cauchy", {"sigma": 1.0}, w)
    assert fkt.relativeError(zd, zdr) <= 1e-13
    assert abs(fkt.relativeError(z, zdr) - 3.42e-4) < 0.1e-4


KERNELS = [
    ("exponential", {}), ("matern12", {"sigma": 1.3, "rho": 0.7}), ("matern32", {"sigma": 0.9, "rho": 0.4}),
    ("cauchy", {"sigma": 0.8}), ("rational-quadratic", {"sigma": 1.1}), ("gaussian", {}), ("inverse-r", {}),
    ("inverse-r2", {}), ("inverse-r3", {}), ("exp-over-r", {}), ("r-exp", {}), ("cos-over-r", {}),
    ("exp-neg-inv-r", {}), ("exp-neg-inv-r2", {}),
]


@pytest.mark.parametrize("name,params", KERNELS)
@pytest.mark.parametrize("d", [2, 3, 5])
def test_kernels_small(fkt, ref, name, params, d):
    x, y = fkt.synthCloud("sphere" if d == 3 else "cube", 3000, d, 7)
    opts = fkt.FktOptions(p=4, theta=0.75, leafCapacity=128)
    p = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, params), opts)
    rp = ref.RefPlan(x, name, params, p=4, theta=0.75, leaf=128)
    assert p.compressed() == rp.compressed
    assert p.coefficientCount() == rp.coef
    z, zr = p.multiply(y), rp.multiply(y)
    assert fkt.relativeError(z, zr) <= TOL


@pytest.mark.parametrize("d,p", [(2, 6), (3, 4), (3, 6), (3, 8), (4, 4), (5, 4), (2, 3), (3, 2), (4, 2), (6, 2),
                                 (3, 0), (2, 1), (3, 1), (5, 2), (2, 10), (3, 10)])
@pytest.mark.parametrize("compression", [1, 2])
def test_orders_dims(fkt, ref, d, p, compression):
    x, y = fkt.synthCloud("mixture", 2500, d, 11)
    opts = fkt.FktOptions(p=p, theta=0.6, leafCapacity=100, compression=fkt.CompressionMode(compression))
    k = fkt.makeKernel("gaussian")
    pl = fkt.plan(fkt.PointCloud.from_array(x), k, opts)
    rp = ref.RefPlan(x, "gaussian", {}, p=p, theta=0.6, leaf=100, compression=compression)
    assert pl.coefficientCount() == rp.coef
    assert fkt.relativeError(pl.multiply(y), rp.multiply(y)) <= TOL


@pytest.mark.parametrize("name,params", KERNELS)
def test_kernels_sixteen_rhs(fkt, ref, name, params):
    # 16 right-hand sides through every kernel's multi-RHS paths (RHS-blocked
    # P2M, tensor-core M2T incl. the runtime-kernel instantiation, 16-RHS
    # near field): each column against the reference's single-RHS multiply
    x, y = fkt.synthCloud("sphere", 4000, 3, 9)
    W = np.stack([np.roll(y, 13 * r) * (1.0 + 0.05 * r) for r in range(16)], axis=1)
    opts = fkt.FktOptions(p=4, theta=0.75, leafCapacity=128)
    p = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, params), opts)
    rp = ref.RefPlan(x, name, params, p=4, theta=0.75, leaf=128)
    Z = p.multiply(W)
    for c in (0, 5, 15):
        col = np.ascontiguousarray(W[:, c])
        assert fkt.relativeError(Z[:, c], rp.multiply(col)) <= TOL, (c,)
