for c in 2 3 4 5; do
  echo "== pf"; SWEEP_CFG=$c python scripts/sweep_near.py 0
  echo "== nopf"; FKTB_LIB_PATH=lib_variants/nopf/libfkt_cuda.so SWEEP_CFG=$c python scripts/sweep_near.py 0
done
SWEEP_CFG=2 python scripts/sweep_near.py 11 1
