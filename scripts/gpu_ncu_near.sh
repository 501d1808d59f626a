# ncu --set full of the near-field stream kernel at the given configs
# usage: bash scripts/gpu_ncu_near.sh TAG CFG...
TAG=$1; shift
for c in "$@"; do bash scripts/gpu_ncu_cfg.sh $c "near_stream" ${TAG}_cfg$c; done
