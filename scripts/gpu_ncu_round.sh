# Round profile set: the launch list of the default cfg2 command (after its
# plain run), then ncu --set full of the near-field and M2T launches at each
# config (scripts/gpu_ncu_r02.sh). usage: bash scripts/gpu_ncu_round.sh TAG
TAG=$1
mkdir -p gpurun_out/$TAG
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/$TAG/ncu_plain.json 2> gpurun_out/$TAG/ncu_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/$TAG/launches_cfg2.csv $CMD > gpurun_out/$TAG/ncu_launch.log 2>&1
echo "launch list rc=$?"
bash scripts/gpu_ncu_r02.sh $TAG 2 3 4 5
