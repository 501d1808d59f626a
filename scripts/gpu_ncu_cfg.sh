# ncu --set full of one kernel family for a given config (plain run first).
# usage: bash scripts/gpu_ncu_cfg.sh CFG REGEX TAG
mkdir -p gpurun_out
CMD="python bench.py --cfg $1 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_$3.json 2> gpurun_out/ncu_plain_$3.err || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"$2" -c 1 -o /tmp/prof_$3 -f $CMD > gpurun_out/ncu_$3.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_$3.log
ncu -i /tmp/prof_$3.ncu-rep --page details > gpurun_out/prof_$3_details.txt 2>&1
ncu -i /tmp/prof_$3.ncu-rep --page raw --csv > gpurun_out/prof_$3_raw.csv 2>&1
ncu -i /tmp/prof_$3.ncu-rep --page source --csv > gpurun_out/prof_$3_source.csv 2>&1
