# A/B/C... of prebuilt libraries on one box: lib<v>.so for v in $LIBS (repo
# root), interleaved reps (v@VAR=1 runs lib<v>.so with VAR=1 in the env); 1M headline step + one beyond-L2 sweep point
for rep in 1 2 3; do
  for spec in ${LIBS:-base variant}; do
    v=${spec%%@*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*@}
    cp lib$v.so paper_2604_26963_b200/libmars_b200.so
    env $envs timeout 300 python bench.py --steps 30 --warmup 5 --no-kv --no-regimes --no-dropin --advance-ticks 0 \
      --hbm-sweep "${SWEEP:-64000000}" --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
sw=' '.join('%dM scan %.3f ctl %.3f step %.3f' % (r['sessions']//1000000, r['k_scan_ms'], r['k_control_ms'], r['ms_per_step']) for r in d.get('hbm_sweep') or [])
print('$spec', round(d['ms_per_step']*1e3,2), 'min', round(d['step_ms_min']*1e3,2), {k: round(x*1e3,1) for k,x in d['kernel_ms_median'].items()}, sw)"
  done
done
