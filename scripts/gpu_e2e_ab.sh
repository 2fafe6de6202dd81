# e2e A/B: one vs two upload streams (MARS_UP_STREAMS), async upload path
set -x
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for rep in 1 2; do
for v in 1 2; do
  MARS_UP_STREAMS=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-kv --no-regimes --no-dropin --advance-ticks 0 \
    --hbm-sweep "" --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('streams $v', 'step', round(d['ms_per_step']*1e3,2), 'e2e', d['e2e'], 'res', round(d['e2e_resident']['ms_per_step'],4))"
done
done
