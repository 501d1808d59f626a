"""The monomial-moment S2M (leaf P2M + exact M2M shifts + per-node basis
change, csrc/moments.cu) must give the same node moments as the direct
per-node evaluation of the reference's s2m rows (expansion.cpp:263-312):
compared through z, against the direct path (FKTB_S2M=direct, run in a child
process) and against the reference."""
import json
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
kind, n, d, name, p, comp, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), int(sys.argv[6]), sys.argv[7]
x, y = fkt.synthCloud(kind, n, d, 9)
W = np.stack([y, np.roll(y, 7), -y]).T.copy()
pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name), fkt.FktOptions(p=p, theta=0.5, leafCapacity=128, compression=fkt.CompressionMode(comp)))
np.save(out, np.concatenate([pl.multiply(y)[:, None], pl.multiply(W)], axis=1))
""" % ROOT

SHAPES = [("cube", 20000, 3, "cauchy", 6, 0), ("cube", 20000, 3, "gaussian", 4, 1), ("sphere", 30000, 3, "inverse-r", 8, 0),
          ("mixture", 20000, 5, "gaussian", 4, 0), ("mixture", 20000, 2, "cauchy", 6, 0),
          ("cube", 20000, 3, "exponential", 8, 2)]


@pytest.mark.parametrize("kind,n,d,name,p,comp", SHAPES)
def test_moments_path_equals_direct_path(tmp_path, kind, n, d, name, p, comp):
    outs = {}
    for mode in ("moments", "direct"):
        env = dict(os.environ)
        if mode == "direct":
            env["FKTB_S2M"] = "direct"
        f = str(tmp_path / f"{mode}.npy")
        subprocess.run([sys.executable, "-c", CHILD, kind, str(n), str(d), name, str(p), str(comp), f], env=env,
                       check=True, timeout=600)
        outs[mode] = np.load(f)
    a, b = outs["moments"], outs["direct"]
    # column 0 is the single-RHS multiply: with the moment path a Gaussian /
    # Matern-3/2 plan runs the Cartesian M2T there (the direct path keeps the
    # harmonic one), ~1e-12 apart for the compressed Gaussian
    for c in range(a.shape[1]):
        assert np.linalg.norm(a[:, c] - b[:, c]) / np.linalg.norm(b[:, c]) <= (5e-12 if c == 0 else 1e-12)


def test_moments_path_matches_reference(fkt, ref):
    x, y = fkt.synthCloud("sphere", 20000, 3, 4)
    for name, p, comp in [("inverse-r", 8, 0), ("gaussian", 6, 1), ("matern32", 6, 0)]:
        prm = {"sigma": 1.0, "rho": 0.2} if name == "matern32" else {}
        pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(name, prm),
                      fkt.FktOptions(p=p, theta=0.5, leafCapacity=256, compression=fkt.CompressionMode(comp)))
        rp = ref.RefPlan(x, name, prm, p=p, theta=0.5, leaf=256, compression=comp)
        assert fkt.relativeError(pl.multiply(y), rp.multiply(y)) <= 1e-10
