for c in 2 3; do echo "cfg$c base"; SWEEP_CFG=$c python scripts/sweep_near.py 0; done
cp paper_2106_04487_b200/lib/libfkt_cuda.so /tmp/base.so
cp paper_2106_04487_b200/lib_variants/exp9/libfkt_cuda.so paper_2106_04487_b200/lib/libfkt_cuda.so
for c in 2 3; do echo "cfg$c exp9"; SWEEP_CFG=$c python scripts/sweep_near.py 0; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_reference_suite.py -q -x 2>&1 | tail -3
cp /tmp/base.so paper_2106_04487_b200/lib/libfkt_cuda.so
