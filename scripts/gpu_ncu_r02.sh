# ncu --set full of the MVM's near-field and M2T kernels at each config
# (plain run first; one ncu process at a time). Raw CSVs come back in
# gpurun_out/ and scripts/ncu_summary.py turns them into profiles/ncu_near.json.
# usage: bash scripts/gpu_ncu_r02.sh TAG CFG...
TAG=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  CMD="python bench.py --cfg $c --steps 1 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/ncu_plain_${TAG}_cfg$c.json 2> gpurun_out/ncu_plain_${TAG}_cfg$c.err || { echo "plain run cfg$c failed"; continue; }
  ncu --set full --import-source on --clock-control none -k regex:"near_stream|near_kernel|m2t_" -c 3 \
      -o /tmp/prof_${TAG}_cfg$c -f $CMD > gpurun_out/ncu_${TAG}_cfg$c.log 2>&1
  echo "cfg$c ncu rc=$?"
  ncu -i /tmp/prof_${TAG}_cfg$c.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_cfg${c}_raw.csv 2>&1
  ncu -i /tmp/prof_${TAG}_cfg$c.ncu-rep --page details > gpurun_out/prof_${TAG}_cfg${c}_details.txt 2>&1
  ncu -i /tmp/prof_${TAG}_cfg$c.ncu-rep --page source --csv -k regex:near_stream > gpurun_out/prof_${TAG}_cfg${c}_near_source.csv 2>&1
done
