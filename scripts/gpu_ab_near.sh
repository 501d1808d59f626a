# A/B of the near-field variants on cfg2/cfg3 (env knobs), then the bench for all configs.
set -x
for c in 2 3; do
  FKTB_NEAR_GRAM=0 python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_nogram_cfg$c.json 2> gpurun_out/ab_nogram_cfg$c.err
  python -c "import json; d=json.load(open('gpurun_out/ab_nogram_cfg$c.json')); print('nogram', $c, d['stage_ms'], d['parity'])"
done
