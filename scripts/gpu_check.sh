timeout 1200 python -m pytest tests/test_gpu_moments.py tests/test_gpu_parity.py -q -x 2>&1 | tail -4
for c in 2 3 4 5; do python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err; tail -2 gpurun_out/b$c.err; python -c "
import json; d=json.load(open('gpurun_out/b$c.json')); print($c, round(d['value'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity']['rel_l2_vs_reference_fkt'])"; done
