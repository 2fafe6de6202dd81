set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2> gpurun_out/ncu1.err; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_walk|k_compact|k_admit_apply|k_lsd_scatter" -s 10 -c 10 -o gpurun_out/prof_r01 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2> gpurun_out/ncu2.err; echo "ncu full rc=$?"
ls -la gpurun_out
