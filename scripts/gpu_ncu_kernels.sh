# one ncu --set full capture per MVM kernel of the cfg2 bench (plain run first)
mkdir -p gpurun_out
TAG=${1:-r01_v3}; shift
CMD="python bench.py --cfg ${CFG:-2} --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err || { echo "plain run failed"; exit 1; }
for K in ${@:-near_fast m2t_fused p2m_regs to_coef_gemm}; do
  ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -o /tmp/prof_${TAG}_$K -f $CMD > gpurun_out/ncu_full_$K.log 2>&1
  echo "$K rc=$?"
  ncu -i /tmp/prof_${TAG}_$K.ncu-rep --page details > gpurun_out/prof_${TAG}_${K}_details.txt 2>&1
  ncu -i /tmp/prof_${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_${K}_raw.csv 2>&1
  ncu -i /tmp/prof_${TAG}_$K.ncu-rep --page source --csv > gpurun_out/prof_${TAG}_${K}_source.csv 2>&1
done
