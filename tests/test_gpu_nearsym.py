"""The opt-in symmetric near field (FKTB_NEAR_SYM=1, csrc/nearsym.cu) must give
the same z as the one-way near field (transform.cpp:163-181 restated in
csrc/near.cu), up to FP64 atomic ordering: both run in child processes."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2106_04487_b200 as fkt
kind, n, d, name, leaf, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), sys.argv[6]
x, y = fkt.synthCloud(kind, n, d, 5)
W = np.stack([y, np.roll(y, 3)]).T.copy()
pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name), fkt.FktOptions(p=4, theta=0.5, leafCapacity=leaf))
np.save(out, np.concatenate([pl.multiply(y)[:, None], pl.multiply(W)], axis=1))
""" % ROOT

SHAPES = [("cube", 30000, 3, "matern32", 256), ("sphere", 20000, 3, "inverse-r", 128), ("mixture", 20000, 5, "gaussian", 128),
          ("cube", 20000, 2, "cauchy", 64), ("mixture", 5000, 3, "exponential", 512)]


@pytest.mark.parametrize("kind,n,d,name,leaf", SHAPES)
def test_symmetric_near_equals_one_way(tmp_path, kind, n, d, name, leaf):
    outs = {}
    for mode in ("0", "1"):
        env = dict(os.environ, FKTB_NEAR_SYM=mode)
        f = str(tmp_path / f"sym{mode}.npy")
        subprocess.run([sys.executable, "-c", CHILD, kind, str(n), str(d), name, str(leaf), f], env=env, check=True,
                       timeout=600)
        outs[mode] = np.load(f)
    a, b = outs["1"], outs["0"]
    for c in range(a.shape[1]):
        assert np.linalg.norm(a[:, c] - b[:, c]) / np.linalg.norm(b[:, c]) <= 1e-13
