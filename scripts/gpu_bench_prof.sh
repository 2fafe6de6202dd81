# the default bench line + the ncu launch list and one full capture of the step kernels
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-kv --e2e-steps 1 --advance-ticks 0 --hbm-sweep "" --clock-load 0 --no-regimes --no-dropin > /dev/null 2> gpurun_out/ncu_list.err; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_walk|k_control|k_pack|k_kv" -s 12 -c 6 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-kv --e2e-steps 1 --advance-ticks 0 --hbm-sweep "" --clock-load 0 --no-regimes --no-dropin > /dev/null 2> gpurun_out/ncu_full.err; echo "ncu full rc=$?"
