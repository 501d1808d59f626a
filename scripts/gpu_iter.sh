timeout 900 python -m pytest tests -m gpu -q -x -k "near or parity or reference_suite or full or fp32" 2>&1 | tail -3
bash scripts/gpu_bench_all.sh 2>&1 | tail -5
SWEEP_CFG=2 python scripts/sweep_near.py 0 3 11 1 8
SWEEP_CFG=3 python scripts/sweep_near.py 0 8 12 5
