timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for c in 2 4; do for v in 0 8; do echo "cfg$c m2t variant $v"; SWEEP_CFG=$c FKTB_M2T_VARIANT=$v python scripts/sweep_near.py 0; done; done
for c in 1 2 3 4 5; do python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err; python -c "
import json; d=json.load(open('gpurun_out/b$c.json')); print($c, round(d['value'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity']['rel_l2_vs_reference_fkt'])"; done
