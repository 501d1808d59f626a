for c in 5; do echo "cfg$c"; SWEEP_CFG=$c python scripts/sweep_near.py 0; done
timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_reference_suite.py tests/test_gpu_parity.py -q -x -k "rhs or cfg5 or multi or parity" 2>&1 | tail -3
