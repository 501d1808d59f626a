timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -2 gpurun_out/bench8.err
python -c "
import json; d=json.load(open('gpurun_out/bench8.json'))
print(d['value'], d['ms_per_step'], d['stage_ms'], d['roofline']['frac'], d['parity'])"
