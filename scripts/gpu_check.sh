for c in 5 2; do echo "cfg$c $(SWEEP_CFG=$c python scripts/sweep_near.py 0)"; done
timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_full.py -q -x 2>&1 | tail -2
