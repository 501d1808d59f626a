# One ncu --set full capture of the cfg2 MVM kernels (plain run first); the
# report is exported to text on the box (the .ncu-rep itself is too large).
mkdir -p gpurun_out
TAG=${1:-cfg2_v3}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"near_fast|m2t_fused|to_coef|p2m_regs" -c 4 -o /tmp/prof_$TAG -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_full.log
ncu -i /tmp/prof_$TAG.ncu-rep --page details > gpurun_out/prof_${TAG}_details.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv -k regex:near_fast > gpurun_out/prof_${TAG}_near_source.csv 2>&1
