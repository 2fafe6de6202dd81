# quick: smoke + step/reclaim parity + a short bench line (headline + sweep)
set -x
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1500 python -m pytest ${PYTEST_FILES:-tests/test_gpu_step.py tests/test_gpu_reclaim.py} -m gpu -q -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -6
timeout 900 python bench.py --steps 20 --warmup 5 --no-regimes --no-kv --no-dropin --no-cpu-baseline --clock-load 20 ${BENCH_ARGS:-} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("ms_per_step", round(d["ms_per_step"],4), "min", round(d["step_ms_min"],4), "frac", round(d["roofline"]["frac"],4), "e2e_ms", round(d["e2e"]["ms_per_step"],3))
print("kernels", {k: round(v*1e3,1) for k, v in d["kernel_ms_median"].items()})
for r in d.get("hbm_sweep") or []:
    print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
PY
