# k_pack grid sizing: the 1M bench step for several MARS_PACK_CTAS values
for pc in 20 24 28 20 24 28; do
  MARS_PACK_CTAS=$pc timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-kv --hbm-sweep "" \
    --e2e-steps 1 --advance-ticks 0 > gpurun_out/bp_$pc.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bp_$pc.json').read().strip().splitlines()[-1])
print('pack_ctas=$pc', round(d['ms_per_step']*1000,1), 'us min', round(d['step_ms_min']*1000,1), {k: round(v*1000,1) for k,v in d['kernel_ms_median'].items()})"
done
