# Round profile set for cfg2: default bench line (with cpu_baseline), the
# reference arm, the ncu launch list, and one ncu --set full capture of the
# MVM kernels (each ncu pass only after the plain command exited 0).
mkdir -p gpurun_out
TAG=${1:-r01_v3}
python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err || { echo "bench failed"; tail gpurun_out/bench_default_$TAG.err; exit 1; }
cat gpurun_out/bench_default_$TAG.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err; cat gpurun_out/bench_reference_$TAG.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_$TAG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"near_fast|m2t_fused|to_coef|p2m_regs|m2m" -c 5 -o /tmp/prof_$TAG -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full.log
ncu -i /tmp/prof_$TAG.ncu-rep --page details > gpurun_out/prof_${TAG}_details.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv -k regex:near_fast > gpurun_out/prof_${TAG}_near_source.csv 2>&1
