python scripts/sweep_near.py 0
FKTB_M2T_VARIANT=1 python scripts/sweep_near.py 0
for c in 3 4; do SWEEP_CFG=$c python scripts/sweep_near.py 0; SWEEP_CFG=$c FKTB_M2T_VARIANT=1 python scripts/sweep_near.py 0; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
