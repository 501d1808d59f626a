"""GPU: API edge cases beyond the reference suite -- multi-RHS counts that are
not multiples of the kernels' RHS blocking, device multiplies with fresh
buffers on every call (bounded CUDA-graph cache), several plans alive on
one device, and a plan used from two threads (multiply is serialised)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nrhs", [2, 5, 17, 40])
def test_multi_rhs_counts(fkt, nrhs):
    x, y = fkt.synthCloud("mixture", 30000, 2, 4)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("cauchy", {"sigma": 1.0}),
                  fkt.FktOptions(p=6, theta=0.75, leafCapacity=256))
    rng = np.random.default_rng(nrhs)
    Y = rng.standard_normal((30000, nrhs))
    Z = pl.multiply(Y)
    for c in {0, nrhs // 2, nrhs - 1}:
        assert fkt.relativeError(Z[:, c], pl.multiply(Y[:, c])) <= 1e-13


def test_fresh_device_buffers_every_call(fkt):
    import torch

    x, y = fkt.synthCloud("cube", 40000, 3, 6)
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel("matern32", {"sigma": 1.0, "rho": 0.1}),
                  fkt.FktOptions(p=6, theta=0.5, leafCapacity=256))
    z0 = pl.multiply(y)
    st = torch.cuda.Stream()
    for _ in range(24):  # > the plan's graph-cache bound (8)
        yd = torch.from_numpy(y).cuda()
        zd = pl.multiply_device(yd, stream=st)
        st.synchronize()
        assert fkt.relativeError(zd.cpu().numpy(), z0) <= 1e-14


def test_several_plans_and_threads(fkt):
    x, y = fkt.synthCloud("sphere", 30000, 3, 7)
    cl = fkt.PointCloud.from_array(x)
    plans = [fkt.plan(cl, fkt.makeKernel(k), fkt.FktOptions(p=4, leafCapacity=256)) for k in ("inverse-r", "gaussian")]
    ref = [p.multiply(y) for p in plans]
    errs = []

    def work(p, r):
        for _ in range(5):
            errs.append(fkt.relativeError(p.multiply(y), r))

    ts = [threading.Thread(target=work, args=(plans[i % 2], ref[i % 2])) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert len(errs) == 20 and max(errs) <= 1e-14
