# every GPU test without stopping at the first failure (junit + summary in gpurun_out/)
set -x
python __graft_entry__.py smoke 2>&1 | tail -3
timeout ${DEBUG_T:-300} python ${DEBUG_SCRIPT:-scripts/debug_kv_devsim.py} 2>&1 | tail -20
timeout 2400 python -m pytest ${PYTEST_FILES:-tests} -m gpu -q -p no:cacheprovider --durations=15 ${PYTEST_K:+-k "$PYTEST_K"} -rf 2>&1 | tail -60
