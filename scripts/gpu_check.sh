mkdir -p gpurun_out
bash scripts/gpu_bench_all.sh
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
