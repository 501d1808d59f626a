for c in 2 3 4; do echo "cfg$c $(SWEEP_CFG=$c python scripts/sweep_near.py 0)"; done
