"""Tuning sweep (developer tool): time the near-field stage of cfg2 for each
FKTB_NEAR_VARIANT (one subprocess per variant; the knob is read once).

    python scripts/sweep_near.py [variants...]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2106_04487_b200 as fkt
cfg = int(sys.argv[1])
C = {2: ("matern32", {"sigma": 1.0, "rho": 0.1}, 1000000, 6, 512, 0.5),
     5: ("cauchy", {"sigma": 1.0}, 2000000, 6, 512, 0.75),
     3: ("gaussian", {}, 1000000, 4, 1024, 0.75),
     4: ("inverse-r", {}, 4000000, 8, 512, 0.5)}[cfg]
x, w = fkt.synthConfig(cfg, C[2])
p = fkt.plan(fkt.PointCloud.from_array(x), fkt.makeKernel(C[0], C[1]), fkt.FktOptions(p=C[3], theta=C[5], leafCapacity=C[4]))
wc = np.ascontiguousarray(w.T) if w.ndim == 2 else w
nrhs = 1 if w.ndim == 1 else w.shape[1]
y = torch.from_numpy(wc).cuda(); z = torch.empty_like(y)
st = torch.cuda.current_stream()
p.multiply_device(y, z, stream=st)
out = {}
for stage in (1, 2, 3):
    for _ in range(2):
        p.stage_device(stage, y, z, nrhs=nrhs, stream=st)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        p.stage_device(stage, y, z, nrhs=nrhs, stream=st)
    e1.record(st); torch.cuda.synchronize()
    out[stage] = e0.elapsed_time(e1) / 10
print(json.dumps(out))
""" % ROOT


def main():
    cfg = int(os.environ.get("SWEEP_CFG", "2"))
    variants = [int(v) for v in sys.argv[1:]] or [0, 1, 2, 3, 4, 5]
    for v in variants:
        env = dict(os.environ, FKTB_NEAR_VARIANT=str(v))
        res = subprocess.run([sys.executable, "-c", CHILD, str(cfg)], env=env, capture_output=True, text=True)
        line = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else res.stderr[-400:]
        print(f"cfg{cfg} variant {v}: {line}", flush=True)


if __name__ == "__main__":
    main()
