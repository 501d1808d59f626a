# ncu --set full of one kernel regex at one config (plain run first)
# usage: bash scripts/gpu_ncu_one.sh CFG REGEX TAG
mkdir -p gpurun_out
CMD="python bench.py --cfg $1 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > /tmp/plain.json 2> /tmp/plain.err || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"$2" -c 1 -o /tmp/prof_$3 -f $CMD > gpurun_out/ncu_$3.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_$3.ncu-rep --page raw --csv > gpurun_out/prof_$3_raw.csv 2>&1
ncu -i /tmp/prof_$3.ncu-rep --page details > gpurun_out/prof_$3_details.txt 2>&1
ncu -i /tmp/prof_$3.ncu-rep --page source --csv > gpurun_out/prof_$3_source.csv 2>&1
