# k_control grid size vs the whole step (bench timing, graph, L2 flushed)
for per in 512 1024 2048 4096; do
  for rep in 1 2; do
    MARS_CTL_PER_CTA=$per timeout 300 python bench.py --steps 30 --warmup 5 --no-kv --advance-ticks 0 \
      --hbm-sweep "" --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('per=$per', round(d['ms_per_step']*1e3,2), 'min', round(d['step_ms_min']*1e3,2), {k: round(v*1e3,1) for k,v in d['kernel_ms_median'].items()})"
  done
done
