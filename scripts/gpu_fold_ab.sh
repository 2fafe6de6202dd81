# e2e / e2e_resident with the fetch's k_out_fold at several grid sizes (MARS_FOLD_CTAS)
for rep in 1 2 3; do
for v in 64 296 592; do
  MARS_FOLD_CTAS=$v timeout 300 python bench.py --steps 10 --warmup 5 --no-kv --no-regimes --no-dropin --advance-ticks 0 \
    --hbm-sweep "" --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('fold $v', 'step', round(d['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['ms_per_step'],4), 'res', round(d['e2e_resident']['ms_per_step'],4))"
done
done
