# GPU box only: rebuild the library with k_scan phase stamps, print them, and
# run the cooperative-launch micro-benchmark (the box's copy is scratch).
set -x
cd paper_2604_26963_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC -shared -DMARS_PHASE_TIMING -o ../libmars_b200.so \
  mars_kernels.cu mars_kv.cu mars_abi.cu
cd ../..
python scripts/debug_phase_timing.py ${1:-1000000} ${2:-headroom} ${3:-mars} ${4:-} 2>&1
[ -n "$MICRO" ] && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mc scripts/micro_coop.cu && /tmp/mc
