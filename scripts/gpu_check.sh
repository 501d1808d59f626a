for c in 2 3; do for m in 1 2; do echo "cfg$c sym=$m"; FKTB_NEAR_SYM=$m SWEEP_CFG=$c python scripts/sweep_near.py 0; done; done
