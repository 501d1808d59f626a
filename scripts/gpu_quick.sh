# quick iteration: near/parity GPU tests + per-config bench (+ optional SASS-free A/B libs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "near or parity or full or cpp_api" 2>&1 | tail -3
bash scripts/gpu_bench_all.sh 2>&1 | tail -6
python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
import paper_2106_04487_b200 as fkt
a, b = C.c_double(), C.c_double()
for i in range(2):
    fkt._check(fkt.lib.fkt_fp64_peaks(C.byref(a), C.byref(b)))
    print("fp64 peaks: dfma %.2f TF  dmma %.2f TF" % (a.value / 1e12, b.value / 1e12))
PY
