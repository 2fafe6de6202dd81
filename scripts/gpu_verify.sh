# every GPU test, smoke, then a short bench (headline + e2e lines)
set -x
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -8
timeout 400 python bench.py --steps 20 --warmup 5 --no-kv --no-regimes --no-dropin --advance-ticks 0 \
  --hbm-sweep "" --no-cpu-baseline --e2e-steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('step', round(d['ms_per_step']*1e3,2), 'e2e', d['e2e'], 'res', d['e2e_resident'])"
