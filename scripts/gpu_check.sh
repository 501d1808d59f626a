timeout 900 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --near-precision 32 > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; tail -2 gpurun_out/bench_fp32.err
python -c "
import json; d=json.load(open('gpurun_out/bench_fp32.json'))
print(d['value'], d['ms_per_step'], d['stage_ms'], d['parity'])"
