# round-2 baseline: GPU tests, per-config bench lines, FP64 peak probes
mkdir -p gpurun_out
bash scripts/gpu_tests.sh > gpurun_out/tests_r02_base.log 2>&1; tail -4 gpurun_out/tests_r02_base.log
bash scripts/gpu_bench_all.sh 2>&1 | tail -6
python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
import paper_2106_04487_b200 as fkt
a, b = C.c_double(), C.c_double()
for i in range(3):
    fkt._check(fkt.lib.fkt_fp64_peaks(C.byref(a), C.byref(b)))
    print("fp64 peaks: dfma %.2f TF  dmma %.2f TF" % (a.value / 1e12, b.value / 1e12))
PY
