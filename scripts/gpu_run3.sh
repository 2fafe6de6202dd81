set -x
python __graft_entry__.py smoke 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 2>&1 | tail -40
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench2.json; tail -5 gpurun_out/bench2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_walk|k_compact|k_admit_apply|k_pack_small" -s 12 -c 6 -o gpurun_out/prof_r01b python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2> gpurun_out/ncu3.err; echo "ncu full rc=$?"
