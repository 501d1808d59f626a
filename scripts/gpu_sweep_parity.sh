# A/B of variant builds: stage times + z parity vs the reference FKT per config.
# usage: bash scripts/gpu_sweep_parity.sh "CFGS" NAME...
CFGS=$1; shift
for c in $CFGS; do
  for v in base "$@"; do
    if [ "$v" = base ]; then unset FKTB_LIB_PATH; else export FKTB_LIB_PATH=$PWD/lib_variants/$v/libfkt_cuda.so; fi
    python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline > /tmp/sw.json 2>/tmp/sw.err || { echo "$v cfg$c failed"; tail -2 /tmp/sw.err; continue; }
    python -c "
import json; d=json.load(open('/tmp/sw.json'))
print('cfg$c', '$v'.ljust(10), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'z_vs_ref %.3e' % d['parity']['rel_l2_vs_reference_fkt'])"
  done
done
unset FKTB_LIB_PATH
