# end-of-round measurements: the default bench line, its ncu launch list and
# one full capture of the step kernels (each after the plain run exited 0)
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
NCU_ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-kv --no-regimes --no-dropin --e2e-steps 1 --advance-ticks 0 --hbm-sweep '' --clock-load 0"
eval timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches.csv python bench.py $NCU_ARGS > /dev/null 2> gpurun_out/ncu_list.err; echo "ncu list rc=$?"
eval timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:"k_scan|k_walk|k_control|k_pack|k_kv_exp_push|k_kv_apply_step|k_out_fold"' -s 16 -c 7 -o gpurun_out/prof python bench.py $NCU_ARGS > /dev/null 2> gpurun_out/ncu_full.err; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.err
