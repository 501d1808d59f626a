for c in 2 3; do
  echo "== default"; SWEEP_CFG=$c python scripts/sweep_near.py 0 1 3 5 8 10 12
  echo "== nogram"; FKTB_NEAR_GRAM=0 SWEEP_CFG=$c python scripts/sweep_near.py 0
  for v in bits9 nofi; do echo "== $v"; FKTB_LIB_PATH=lib_variants/$v/libfkt_cuda.so SWEEP_CFG=$c python scripts/sweep_near.py 0; done
done
