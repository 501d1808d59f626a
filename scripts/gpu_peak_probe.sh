nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
./scripts/probes/dmma_probe
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
python - <<'PY'
import ctypes as C, sys, time, subprocess
sys.path.insert(0, ".")
import paper_2106_04487_b200 as fkt
a, b = C.c_double(), C.c_double()
for i in range(3):
    fkt._check(fkt.lib.fkt_fp64_peaks(C.byref(a), C.byref(b)))
    print("fp64 peaks: dfma %.2f TF  dmma %.2f TF" % (a.value / 1e12, b.value / 1e12), flush=True)
    time.sleep(2)
PY
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/peak_clocks.csv & SMI=$!; sleep 0.5
./scripts/probes/dmma_probe
sleep 0.5; kill $SMI; sort gpurun_out/peak_clocks.csv | uniq -c | sort -rn | head
