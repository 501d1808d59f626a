# deterministic mode: GPU tests (+ the whole GPU suite) and bench lines with it
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_deterministic.py -q -x 2>&1 | tail -15
for c in 2 5 4; do
  python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline --deterministic > gpurun_out/bench_det_cfg$c.json 2> gpurun_out/bench_det_cfg$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_det_cfg$c.json'))
print('det', $c, round(d['value'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity'], round(d['config']['plan_seconds'],3))" || tail -5 gpurun_out/bench_det_cfg$c.err
done
${FULL:+bash scripts/gpu_tests.sh > gpurun_out/tests_det.log 2>&1; tail -4 gpurun_out/tests_det.log}
