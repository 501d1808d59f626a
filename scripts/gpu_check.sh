timeout 1200 python -m pytest tests/test_gpu_barnes_hut.py tests/test_gpu_distributed.py tests/test_gpu_reference_suite.py -q -x 2>&1 | tail -15
