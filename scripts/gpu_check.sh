timeout 900 python -m pytest tests/test_gpu_nearsym.py -q -x 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -1
