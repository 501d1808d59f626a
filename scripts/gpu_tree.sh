# tree/sets parity (reference suite + full-size fingerprints) and plan timings
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_parity.py tests/test_gpu_full.py -q -x 2>&1 | tail -3
for c in 1 2 3 4 5; do
  python bench.py --cfg $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tree_cfg$c.json 2> gpurun_out/bench_tree_cfg$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_tree_cfg$c.json')); c=d['config']
print($c, round(d['value'],2), 'plan', round(c['plan_seconds']*1e3,1), 'replan', round(c['replan_seconds']*1e3,1), {k: round(v*1e3,1) for k,v in c['replan_phases'].items()})" || tail -3 gpurun_out/bench_tree_cfg$c.err
done
