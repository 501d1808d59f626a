for c in 2 3 4 5; do echo "cfg$c"; SWEEP_CFG=$c python scripts/sweep_near.py 0; done
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_full.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -3
