for c in 1 2 3 4 5; do
  python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_cfg$c.json'))
print($c, round(d['value'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['frac'],3), d['parity'], round(d['config']['plan_seconds'],3))"
done
