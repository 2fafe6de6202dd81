set -x
timeout 1500 python -m pytest tests/test_gpu_kv.py tests/test_gpu_devsim.py tests/test_gpu_ticks.py -m gpu -q -p no:cacheprovider -x -k "block_ids or kv or fuzz or journal or deep or scale or ticks" 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_s5.csv python scripts/prof_scan.py 1000000 s5 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/l_s5.csv')))
h=None
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        if d.get('Metric Name')=='gpu__time_duration.sum': print(d['Kernel Name'][:40], d['Metric Value'])
PY
timeout 900 python bench.py --steps 20 --warmup 5 --hbm-sweep "" --no-regimes --no-kv --no-dropin --no-cpu-baseline --clock-load 20 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("ms_per_step", round(d["ms_per_step"],4), "min", round(d["step_ms_min"],4), "frac", round(d["roofline"]["frac"],4), "e2e_ms", round(d["e2e"]["ms_per_step"],3))
print("kernels", {k: round(v*1e3,1) for k, v in d["kernel_ms_median"].items()})
PY
