# ncu --set full of the cfg2 near kernel for the given FKTB_NEAR_VARIANT values
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err || { echo "plain run failed"; exit 1; }
for V in "$@"; do
  FKTB_NEAR_VARIANT=$V ncu --set full --import-source on --clock-control none -k regex:"near_fast" -c 1 -o /tmp/prof_near_v$V -f $CMD > gpurun_out/ncu_near_v$V.log 2>&1
  echo "v$V rc=$?"
  ncu -i /tmp/prof_near_v$V.ncu-rep --page details > gpurun_out/prof_near_v${V}_details.txt 2>&1
  ncu -i /tmp/prof_near_v$V.ncu-rep --page raw --csv > gpurun_out/prof_near_v${V}_raw.csv 2>&1
  ncu -i /tmp/prof_near_v$V.ncu-rep --page source --csv > gpurun_out/prof_near_v${V}_source.csv 2>&1
done
