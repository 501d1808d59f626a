for c in 2 4 5; do
  echo "== atomics"; SWEEP_CFG=$c python scripts/sweep_near.py 0
  echo "== no atomics (timing only)"; FKTB_LIB_PATH=lib_variants/noatom/libfkt_cuda.so SWEEP_CFG=$c python scripts/sweep_near.py 0
done
