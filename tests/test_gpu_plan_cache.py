"""GPU: the plan cache (fkt_plan_cache_*): identical requests
share one device plan, different inputs do not, unreferenced plans are kept
up to the capacity and evicted LRU, and cached plans multiply exactly like
fresh ones."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_plan_cache(fkt):
    x, y = fkt.synthCloud("cube", 50000, 3, 3)
    cl = fkt.PointCloud.from_array(x)
    k = fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.1})
    o = fkt.FktOptions(p=6, theta=0.5, leafCapacity=256)
    fkt.planCacheCapacity(2)
    a = fkt.cachedPlan(cl, k, o)
    b = fkt.cachedPlan(cl, k, o)
    assert not a.cacheHit and b.cacheHit and a._h.value == b._h.value
    z = fkt.plan(cl, k, o).multiply(y)
    assert fkt.relativeError(b.multiply(y), a.multiply(y)) <= 1e-15  # FP64 atomics: roundoff-equal
    assert fkt.relativeError(a.multiply(y), z) <= 1e-14
    # any difference in cloud, kernel parameters or options is a miss
    x2 = x.copy()
    x2[7, 1] = np.nextafter(x2[7, 1], 2.0)
    assert not fkt.cachedPlan(fkt.PointCloud.from_array(x2), k, o).cacheHit
    assert not fkt.cachedPlan(cl, fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.11}), o).cacheHit
    assert not fkt.cachedPlan(cl, k, fkt.FktOptions(p=6, theta=0.5, leafCapacity=256, nearPrecision=32)).cacheHit
    # released plans stay cached up to the capacity (2): the two newest survive
    del a, b
    import gc

    gc.collect()
    assert fkt.planCacheSize() == 2  # the shared plan and the newest miss (nearPrecision 32)
    assert fkt.cachedPlan(cl, k, o).cacheHit  # touched: now the most recent
    assert not fkt.cachedPlan(cl, fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.12}), o).cacheHit
    assert fkt.planCacheSize() == 2  # the nearPrecision-32 plan was least recently used: evicted
    assert not fkt.cachedPlan(cl, k, fkt.FktOptions(p=6, theta=0.5, leafCapacity=256, nearPrecision=32)).cacheHit
    # a cached plan cannot be destroyed directly
    c = fkt.cachedPlan(cl, k, o)
    assert fkt.lib.fkt_plan_destroy(c._h) == 1  # FKT_ERR_INVALID_ARGUMENT
    del c
    gc.collect()
    fkt.planCacheCapacity(0)
    assert fkt.planCacheSize() == 0
    fkt.planCacheCapacity(4)
