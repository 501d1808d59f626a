timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
mkdir -p gpurun_out
bash scripts/gpu_bench_all.sh
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
