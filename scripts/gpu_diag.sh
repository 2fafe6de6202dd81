# diagnostics: e2e breakdown, drop-in host profile, k_scan/step phase stamps (writes gpurun_out/)
set -x
timeout 300 python scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; tail -20 gpurun_out/e2e_breakdown.txt
timeout 300 python scripts/prof_dropin.py > gpurun_out/prof_dropin.txt 2>&1; head -60 gpurun_out/prof_dropin.txt
timeout 600 bash scripts/gpu_phase_timing.sh 1000000 headroom mars s5 > gpurun_out/phase.txt 2>&1; tail -60 gpurun_out/phase.txt
