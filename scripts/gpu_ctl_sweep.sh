# k_control grid sizing sweep: phase stamps of the LSD pack sort at 1M sessions
cd paper_2604_26963_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC -shared -DMARS_PHASE_TIMING -o ../libmars_b200.so \
  mars_kernels.cu mars_kv.cu mars_abi.cu 2>/dev/null
cd ../..
for per in 1024 2048 4096; do
  echo "=== MARS_CTL_PER_CTA=$per"
  MARS_CTL_PER_CTA=$per python scripts/debug_phase_timing.py 2>&1 | grep -A40 "graph step 1" | grep "stamp  [0-9]:\|stamp 1[0-5]\|stamp 2[0-4]\|graph"
done
