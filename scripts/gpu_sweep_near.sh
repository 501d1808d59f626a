# near-field variant sweep (FKTB_NEAR_VARIANT) for cfg2 and cfg3
SWEEP_CFG=2 python scripts/sweep_near.py 0 1 2 3 4 5 6 7 8 9 10 12 13
SWEEP_CFG=3 python scripts/sweep_near.py 0 1 4 5 6 8 9 10 12 13
