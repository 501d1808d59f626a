# tests + per-config bench (+ optional extra command)
bash scripts/gpu_tests.sh > gpurun_out/tests_round.log 2>&1; tail -4 gpurun_out/tests_round.log
bash scripts/gpu_bench_all.sh 2>&1 | tail -5
