# Round-2 measurement set: default bench line (cfg2, cpu_baseline), the
# reference arm (full-size reference MVMs), per-config lines, deterministic and
# FP32 lines, and the ncu launch list of the default command.
TAG=${1:-r02i}
export TAG
mkdir -p gpurun_out/$TAG
python bench.py > gpurun_out/$TAG/bench_default_cfg2.json 2> gpurun_out/$TAG/bench_default_cfg2.err || tail -5 gpurun_out/$TAG/bench_default_cfg2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_reference_cfg2.json 2> gpurun_out/$TAG/bench_reference_cfg2.err
for c in 1 2 3 4 5; do
  python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_cfg$c.json 2> gpurun_out/$TAG/bench_cfg$c.err
  python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline --deterministic > gpurun_out/$TAG/bench_det_cfg$c.json 2> gpurun_out/$TAG/bench_det_cfg$c.err
done
for c in 2 3 5; do
  python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline --near-precision 32 > gpurun_out/$TAG/bench_fp32_cfg$c.json 2> gpurun_out/$TAG/bench_fp32_cfg$c.err
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/$TAG/ncu_plain.json 2> gpurun_out/$TAG/ncu_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/$TAG/launches_cfg2.csv $CMD > gpurun_out/$TAG/ncu_launch.log 2>&1
echo "launch list rc=$?"
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/" + os.environ["TAG"] + "/bench_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    if "value" not in d:
        print(f, d); continue
    print(f.split("/")[-1], round(d["value"], 4), d.get("e2e", {}).get("value"), d.get("parity"))
PY
