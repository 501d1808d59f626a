# ncu evidence for the cfg2 MVM kernels (run under gpurun, 1 GPU).
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"near_fast|m2t_fast|s2m_fast|gather_y|scatter_z" -c 10 --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"near_fast|m2t_fast|s2m_fast" -c 3 -o gpurun_out/prof_cfg2 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full.log
