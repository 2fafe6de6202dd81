# GPU parity tests (subset via PYTEST_FILES / PYTEST_K), then a short bench line
set -x
python __graft_entry__.py smoke 2>&1 | tail -3
timeout 1500 python -m pytest ${PYTEST_FILES:-tests} -m gpu -q -p no:cacheprovider -x --durations=10 ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -40
if [ -n "$BENCH" ]; then
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-kv ${BENCH_ARGS:-} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("ms_per_step", d["ms_per_step"], "min", d["step_ms_min"], "kernels", d["kernel_ms_median"],
      "frac", d["roofline"]["frac"], "e2e_ms", d["e2e"]["ms_per_step"])
for k in ("regimes", "hbm_sweep"):
    v = d.get(k)
    if isinstance(v, list):
        for r in v: print({a: (round(b, 4) if isinstance(b, float) else b) for a, b in r.items()})
    elif v is not None:
        print(k, v)
PY
fi
