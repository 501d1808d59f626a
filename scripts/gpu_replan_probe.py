"""Re-plan timing probe: plan + several rebuilds, phases printed each time."""
import sys
import time

import numpy as np

import paper_2106_04487_b200 as fkt

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402

for cfg in [int(a) for a in sys.argv[1:]] or [2]:
    c = CONFIGS[cfg]
    x, w = fkt.synthConfig(cfg, c["n"])
    t0 = time.perf_counter()
    pl = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(c["kernel"], c["params"]),
                  fkt.FktOptions(p=c["p"], theta=c["theta"], leafCapacity=c["leaf"]))
    print(f"cfg{cfg} plan {time.perf_counter() - t0:.4f}", {k: round(v * 1e3, 2) for k, v in pl.plan_phases().items()}, flush=True)
    rng = np.random.default_rng(3)
    xm = x + 1e-3 * rng.standard_normal(x.shape) * x.std(axis=0)
    for i in range(6):
        t0 = time.perf_counter()
        pl.rebuild(xm if i % 2 == 0 else x)
        print(f"cfg{cfg} rebuild{i} {1e3 * (time.perf_counter() - t0):.2f} ms", {k: round(v * 1e3, 2) for k, v in pl.plan_phases().items()}, flush=True)
    del pl
