"""GPU: re-planning for moving points (FktPlan.rebuild / fkt_plan_rebuild).

t-SNE-style uses move the points every iteration; the reference rebuilds the
whole FktPlan from the new PointCloud (transform.cpp:39-92). The rebuild keeps
the plan's kernel tables and buffers and must give exactly what a fresh plan
on the new points gives: bit-identical tree and interaction sets, and (in
deterministic mode) bitwise-identical z."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _fresh(fkt, x, name, prm, **kw):
    return fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm), fkt.FktOptions(**kw))


def _same_tree(a, b):
    ta, tb = a.tree(), b.tree()
    np.testing.assert_array_equal(ta.order(), tb.order())
    np.testing.assert_array_equal(ta.begins, tb.begins)
    np.testing.assert_array_equal(ta.lefts, tb.lefts)
    np.testing.assert_array_equal(ta.radii.view(np.uint64), tb.radii.view(np.uint64))
    for csr in ("farCsr", "nearCsr"):
        oa, ia = getattr(ta, csr)()
        ob, ib = getattr(tb, csr)()
        np.testing.assert_array_equal(oa, ob)
        np.testing.assert_array_equal(ia, ib)


CASES = [("cube", 60000, 3, "matern32", {"sigma": 1.0, "rho": 0.1}, dict(p=6, theta=0.5, leafCapacity=256)),
         ("mixture", 80000, 2, "cauchy", {"sigma": 1.0}, dict(p=6, theta=0.75, leafCapacity=512)),
         ("sphere", 50000, 3, "inverse-r", {}, dict(p=8, theta=0.5, leafCapacity=256)),
         ("cube", 30000, 3, "exponential", {}, dict(p=5, theta=0.6, leafCapacity=128)),  # generic (d, p)
         ("sphere", 40000, 3, "inverse-r", {}, dict(p=0, theta=0.5, leafCapacity=128, barnesHut=True))]


@pytest.mark.parametrize("kind,n,d,name,prm,kw", CASES)
def test_rebuild_equals_fresh_plan(fkt, kind, n, d, name, prm, kw):
    x0, y = fkt.synthCloud(kind, n, d, 31)
    rng = np.random.default_rng(4)
    pl = _fresh(fkt, x0, name, prm, deterministic=True, **kw)
    x = x0
    for it in range(3):  # moving points: small steps, then a jump
        x = x + (0.02 if it < 2 else 0.5) * rng.standard_normal(x.shape) * x.std(axis=0)
        pl.rebuild(x)
        fresh = _fresh(fkt, x, name, prm, deterministic=True, **kw)
        _same_tree(pl, fresh)
        assert pl.coefficientCount() == fresh.coefficientCount()
        z1, z2 = pl.multiply(y), fresh.multiply(y)
        assert np.array_equal(z1, z2), f"iteration {it}: rebuilt plan differs from a fresh plan"
        del fresh


def test_rebuild_matches_reference(fkt, ref):
    x0, y = fkt.synthConfig(1, 20000)
    pl = _fresh(fkt, x0, "cauchy", {"sigma": 1.0}, p=4, theta=0.5, leafCapacity=512)
    x = x0[::-1].copy() * 1.3 + 0.1  # new geometry, same n
    pl.rebuild(x)
    rp = ref.RefPlan(x, "cauchy", {"sigma": 1.0}, p=4, theta=0.5, leaf=512)
    np.testing.assert_array_equal(pl.tree().order(), rp.tree()["order"])
    assert fkt.relativeError(pl.multiply(y), rp.multiply(y)) <= 1e-10


def test_rebuild_sharded_and_device_path(fkt):
    import torch

    x0, y = fkt.synthCloud("cube", 50000, 3, 9)
    pl = _fresh(fkt, x0, "matern32", {"sigma": 1.0, "rho": 0.2}, p=6, theta=0.5, leafCapacity=256)
    yd = torch.from_numpy(y).cuda()
    st = torch.cuda.Stream()
    zd = torch.empty_like(yd)
    pl.multiply_device(yd, zd, stream=st)  # captures a graph on this (y, z, stream)
    x = x0 * 0.7 + 0.2
    pl.rebuild(x)
    pl.multiply_device(yd, zd, stream=st)  # the stale graph must not replay
    st.synchronize()
    fresh = _fresh(fkt, x, "matern32", {"sigma": 1.0, "rho": 0.2}, p=6, theta=0.5, leafCapacity=256)
    zf = fresh.multiply(y)
    assert fkt.relativeError(zd.cpu().numpy(), zf) <= 1e-13
    pl.set_shard(1, 3)
    lo, hi = pl.shard_range()
    pl.rebuild(x0)  # the shard is re-cut on the new tree
    assert pl.shard_range() != (0, 50000)
    pl.set_shard(0, 1)
    assert fkt.relativeError(pl.multiply(y), _fresh(fkt, x0, "matern32", {"sigma": 1.0, "rho": 0.2}, p=6, theta=0.5,
                                                    leafCapacity=256).multiply(y)) <= 1e-13


def test_rebuild_errors(fkt):
    x0, _ = fkt.synthCloud("cube", 5000, 3, 2)
    pl = _fresh(fkt, x0, "cauchy", {}, p=4)
    with pytest.raises(fkt.DimensionMismatchError):
        pl.rebuild(x0[:4000])
    with pytest.raises(fkt.DimensionMismatchError):
        pl.rebuild(np.zeros((5000, 2)))
    cached = fkt.FktPlan(fkt.PointCloud.from_array(x0), fkt.makeKernel("cauchy", {}), fkt.FktOptions(p=4), _cached=True)
    with pytest.raises(fkt.InvalidArgument):
        cached.rebuild(x0)


def test_rebuild_device_equals_host_rebuild(fkt):
    """fkt_plan_rebuild_device: coordinates already in HBM (a t-SNE embedding
    updated on the GPU); same tree, sets and deterministic z as the host-buffer
    rebuild, and cloud() returns the new points."""
    import torch

    x0, y = fkt.synthCloud("mixture", 70000, 2, 5)
    kw = dict(p=6, theta=0.75, leafCapacity=512, deterministic=True)
    a = _fresh(fkt, x0, "cauchy", {"sigma": 1.0}, **kw)
    b = _fresh(fkt, x0, "cauchy", {"sigma": 1.0}, **kw)
    rng = np.random.default_rng(8)
    x = x0
    for it in range(3):
        x = x + 0.05 * rng.standard_normal(x.shape) * x.std(axis=0)
        a.rebuild(x)
        b.rebuild_device(torch.from_numpy(x).cuda())
        _same_tree(a, b)
        assert np.array_equal(a.multiply(y), b.multiply(y))
        np.testing.assert_array_equal(b.cloud().x, x)
    with pytest.raises(fkt.DimensionMismatchError):
        b.rebuild_device(torch.zeros(10, 2, dtype=torch.float64, device="cuda"))
    with pytest.raises(fkt.DimensionMismatchError):
        b.rebuild_device(torch.from_numpy(x.astype(np.float32)).cuda())
