# one GPU session: smoke, GPU parity tests, bench, ncu captures (writes gpurun_out/)
set -x
python __graft_entry__.py smoke 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 -x 2>&1 | tail -30
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
# launch list of the same bench command (per-launch durations, serialised, no profiler cache flush)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-kv --e2e-steps 1 --advance-ticks 0 --hbm-sweep "" --clock-load 0 > /dev/null 2> gpurun_out/ncu_list.err; echo "ncu list rc=$?"
# one full capture of each step kernel (k_scan, k_control, k_walk)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_walk|k_control|k_pack" -s 8 -c 4 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-kv --e2e-steps 1 --advance-ticks 0 --hbm-sweep "" --clock-load 0 > /dev/null 2> gpurun_out/ncu_full.err; echo "ncu full rc=$?"
