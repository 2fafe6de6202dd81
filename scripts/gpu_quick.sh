# quick GPU iteration: step parity tests, a short bench line, then the phase
# timeline of a debug rebuild (the box's copy of the library is scratch)
set -x
timeout 900 python -m pytest ${PYTEST_FILES:-tests/test_gpu_step.py} -q -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-kv ${BENCH_ARGS:-} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("ms_per_step", d["ms_per_step"], "min", d["step_ms_min"], "kernels", d["kernel_ms_median"],
      "frac", d["roofline"]["frac"], "e2e_ms", d["e2e"]["ms_per_step"])
for r in d.get("hbm_sweep") or []:
    print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
PY
bash scripts/gpu_phase_timing.sh 2>&1 | grep -v "^+" | head -75
