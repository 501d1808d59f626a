timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in 2 3 4 5; do SWEEP_CFG=$c python scripts/sweep_near.py 0; done
