# parity subset on the in-tree library, then an A/B of libbase.so vs libvariant.so
set -x
timeout 900 python -m pytest ${PYTEST_FILES:-tests/test_gpu_step.py tests/test_gpu_kv.py tests/test_gpu_reclaim.py} -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
SWEEP=${SWEEP:-16000000} LIBS="${LIBS:-base variant}" bash scripts/ab_multi.sh 2>&1
