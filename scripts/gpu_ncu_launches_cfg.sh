# ncu launch list (per-kernel durations, serialised, cold) of the MVM kernels at the given configs.
# usage: bash scripts/gpu_ncu_launches_cfg.sh "4 5"
mkdir -p gpurun_out
for c in $1; do
  CMD="python bench.py --cfg $c --steps 1 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/ncu_plain_cfg$c.json 2> gpurun_out/ncu_plain_cfg$c.err || { echo "plain run failed cfg$c"; tail -3 gpurun_out/ncu_plain_cfg$c.err; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --kernel-name 'regex:near_stream|near_kernel|near_fill|near_weights|m2t_|s2m_|p2m_|m2m_|to_coef|gather_y|scatter_z|det_|tile_sum' \
      --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_launch_cfg$c.log 2>&1
  echo "cfg$c rc=$?"
done
