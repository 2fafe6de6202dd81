# e2e / e2e_resident A/B of prebuilt libraries (lib<v>.so at the repo root)
for rep in 1 2 3; do
for v in ${LIBS:-base variant}; do
  cp lib$v.so paper_2604_26963_b200/libmars_b200.so
  timeout 300 python bench.py --steps 10 --warmup 5 --no-kv --no-regimes --no-dropin --advance-ticks 0 \
    --hbm-sweep "" --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', 'step', round(d['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['ms_per_step'],4), 'upload', round(d['e2e']['upload_ms'],4), 'res', round(d['e2e_resident']['ms_per_step'],4))"
done
done
