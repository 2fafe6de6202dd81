# A/B two prebuilt libraries on one box: libbase.so vs libvariant.so (repo root)
for rep in 1 2 3; do
  for v in base variant; do
    cp lib$v.so paper_2604_26963_b200/libmars_b200.so
    timeout 300 python bench.py --steps 30 --warmup 5 --no-kv --advance-ticks 0 --hbm-sweep "" \
      --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', round(d['ms_per_step']*1e3,2), 'min', round(d['step_ms_min']*1e3,2), {k: round(x*1e3,1) for k,x in d['kernel_ms_median'].items()})"
  done
done
