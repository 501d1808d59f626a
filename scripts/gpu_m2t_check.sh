# M2T change check: parity subset + per-config stage times
timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_parity.py tests/test_gpu_m2t_mma.py tests/test_gpu_moments.py tests/test_gpu_deterministic.py -q -x 2>&1 | tail -3
for c in 2 5; do
  python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  python -c "
import json; d=json.load(open('/tmp/b.json'))
print('cfg$c', round(d['value'],3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['parity']['rel_l2_vs_reference_fkt'])" || tail -3 /tmp/b.err
done
