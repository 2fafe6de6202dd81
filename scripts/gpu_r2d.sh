set -x
timeout 1500 python -m pytest tests/test_gpu_kv.py tests/test_gpu_sharded.py tests/test_gpu_devsim.py -m gpu -q -p no:cacheprovider -x -k "block_ids or kv or fuzz or journal or deep or scale or sharded or replica" 2>&1 | tail -8
bash scripts/gpu_sharded_bench_check.sh 2>&1 | tail -8
timeout 900 python bench.py --steps 20 --warmup 5 --hbm-sweep "" --no-regimes --no-kv --no-dropin --no-cpu-baseline > gpurun_out/bench_s5.json 2> gpurun_out/bench_s5.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_s5.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_s5.json").read().strip().splitlines()[-1])
print("ms_per_step", d["ms_per_step"], "min", d["step_ms_min"], "frac", d["roofline"]["frac"], "e2e_ms", d["e2e"]["ms_per_step"])
print("kernels", d["kernel_ms_median"])
print("adv", d["advance"]["ms_per_tick"], d["advance"]["ms_per_tick_control"])
PY
