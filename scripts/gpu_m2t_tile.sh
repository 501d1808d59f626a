for t in 1024 2048 4096 8192; do
  for c in 2 4 5; do echo "tile $t"; FKTB_M2T_TILE=$t SWEEP_CFG=$c python scripts/sweep_near.py 0; done
done
