timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in 1 2 5; do python bench.py --cfg $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err; tail -2 gpurun_out/b$c.err; python -c "
import json; d=json.load(open('gpurun_out/b$c.json')); print($c, d['value'], d['ms_per_step'], d['e2e']['value'], d['parity']['rel_l2_vs_reference_fkt'])"; done
