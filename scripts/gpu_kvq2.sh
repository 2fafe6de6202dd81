set -x
for c in 1 default; do if [ $c = default ]; then unset CUDA_DEVICE_MAX_CONNECTIONS; else export CUDA_DEVICE_MAX_CONNECTIONS=$c; fi
timeout 600 python -m pytest tests/test_gpu_kv.py -m gpu -q -p no:cacheprovider -x -k "scale or journal" 2>&1 | tail -2
done
unset CUDA_DEVICE_MAX_CONNECTIONS
timeout 900 python bench.py --steps 20 --warmup 5 --hbm-sweep "" --no-regimes --no-kv --no-dropin --no-cpu-baseline --clock-load 20 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("ms_per_step", round(d["ms_per_step"],4), "min", round(d["step_ms_min"],4), "frac", round(d["roofline"]["frac"],4), "e2e_ms", round(d["e2e"]["ms_per_step"],3), "resident", round(d["e2e_resident"]["ms_per_step"],3))
print("kernels", {k: round(v*1e3,1) for k, v in d["kernel_ms_median"].items()})
PY
