set -x
timeout 300 python scripts/debug_kv_devsim.py 2>&1 | tail -5
timeout 1500 python -m pytest tests/test_gpu_devsim.py tests/test_gpu_kv.py tests/test_gpu_dropin.py tests/test_gpu_realsim.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 900 python bench.py --steps 20 --warmup 5 --hbm-sweep "" --no-regimes --no-kv > gpurun_out/bench_s5.json 2> gpurun_out/bench_s5.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_s5.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_s5.json").read().strip().splitlines()[-1])
print("ms_per_step", d["ms_per_step"], "min", d["step_ms_min"], "frac", d["roofline"]["frac"], "e2e_ms", d["e2e"]["ms_per_step"])
print("kernels", d["kernel_ms_median"])
print("adv", d["advance"])
for r in d.get("dropin", []): print(r)
print("cpu", d.get("cpu_baseline"))
PY
