timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_moments.py -q -x 2>&1 | tail -2
for c in 3 4; do for v in 0 3; do echo "m2t variant $v"; SWEEP_CFG=$c FKTB_M2T_VARIANT=$v python scripts/sweep_near.py 0; done; done
