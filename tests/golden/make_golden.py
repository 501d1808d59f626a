"""Generate the committed golden fixtures from the REFERENCE itself.

Runs in the build container (needs oracle/_ref, i.e. /root/reference at build
time). For every BASELINE config it builds the reference plan on the Appendix B
inputs, runs the reference multiply (streaming, all host cores), and stores:
  * fingerprints (order / sets / geom) and tree counts,
  * z of the reference FKT on 1000 sampled rows (fkt::Rng(7).next() % N),
  * the dense O(N^2) product on the same rows (reference kernel arithmetic),
  * the reference plan / multiply wall times on this box.
cfg1 also stores the full z vector.

    python tests/golden/make_golden.py [cfg ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

CONFIGS = {
    1: dict(kernel="cauchy", params={"sigma": 1.0}, n=20000, p=4, leaf=512, theta=0.5),
    2: dict(kernel="matern32", params={"sigma": 1.0, "rho": 0.1}, n=1000000, p=6, leaf=512, theta=0.5),
    3: dict(kernel="gaussian", params={}, n=1000000, p=4, leaf=1024, theta=0.75),
    4: dict(kernel="inverse-r", params={}, n=4000000, p=8, leaf=512, theta=0.5),
    5: dict(kernel="cauchy", params={"sigma": 1.0}, n=2000000, p=6, leaf=512, theta=0.75),
}


def splitmix_rows(seed: int, count: int, n: int) -> np.ndarray:
    M = (1 << 64) - 1
    state = seed
    out = []
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z = z ^ (z >> 31)
        out.append(z % n)
    return np.array(out, dtype=np.int64)


def main(cfgs):
    here = os.path.dirname(os.path.abspath(__file__))
    for cfg in cfgs:
        c = CONFIGS[cfg]
        t0 = time.time()
        x, w = ref.gen_config(cfg, c["n"])
        rp = ref.RefPlan(x, c["kernel"], c["params"], p=c["p"], theta=c["theta"], leaf=c["leaf"],
                         eager=c["n"] < 100000)
        fp = rp.fingerprints()
        t1 = time.time()
        z = rp.multiply(w)
        t2 = time.time()
        rows = splitmix_rows(7, 1000, c["n"])
        wcol = w if w.ndim == 1 else w[:, 0]
        zcol = z if z.ndim == 1 else z[:, 0]
        dense = ref.dense_rows(x, c["kernel"], c["params"], wcol, rows)
        out = dict(rows=rows, z_rows=(z[rows] if z.ndim == 1 else z[rows, :]), dense_rows=dense)
        if cfg == 1:
            out["z"] = z
        np.savez_compressed(os.path.join(here, f"cfg{cfg}_ref.npz"), **out)
        meta = dict(cfg=cfg, **{k: v for k, v in c.items()}, nodes=rp.nodes, far_total=rp.far_total,
                    near_total=rp.near_total, coef=rp.coef, compressed=rp.compressed, order=fp[0], sets=fp[1],
                    geom=fp[2], plan_s=rp.plan_seconds, mvm_s=t2 - t1, threads=os.cpu_count(),
                    fkt_vs_dense_rows=float(np.linalg.norm(zcol[rows] - dense) / np.linalg.norm(dense)),
                    generated_by="tests/golden/make_golden.py (reference sources via oracle/_ref)")
        with open(os.path.join(here, f"cfg{cfg}_ref.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps(meta), flush=True)
        del rp
        print(f"cfg{cfg} done in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 4])
