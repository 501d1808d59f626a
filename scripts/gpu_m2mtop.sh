for t in 0 6 8 10; do for c in 2 4 5; do
  FKTB_M2M_TOP=$t python bench.py --cfg $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('top', $t, $c, round(d['ms_per_step'],4), round(d['stage_ms']['s2m'],4), d['parity']['rel_l2_vs_reference_fkt'])"
done; done
