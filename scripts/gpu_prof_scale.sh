# ncu captures beyond L2 (16M sessions: k_scan, k_control, k_walk) and of the KV movers
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_control|k_walk" -s 3 -c 3 -o gpurun_out/prof16m python scripts/prof_scan.py 16000000 > gpurun_out/p16.log 2>&1; tail -1 gpurun_out/p16.log
timeout 600 ncu --set full --clock-control none -k regex:"k_kv_stage" -s 2 -c 2 -o gpurun_out/profkv python scripts/prof_kvmove.py > gpurun_out/pkv.log 2>&1; tail -1 gpurun_out/pkv.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_kv_exp_push|k_kv_apply_step" -s 2 -c 2 -o gpurun_out/profs5 python scripts/prof_scan.py 1000000 s5 > gpurun_out/ps5.log 2>&1; tail -1 gpurun_out/ps5.log
