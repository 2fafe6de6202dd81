"""Debug: repeat the kv-only openhands devsim (intermittent status 4 hunt)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from oracle import tracefile
from tests._sim import SIM
from tests.conftest import GOLDEN
from paper_2604_26963_b200.devsim import EventLog, run_device_simulation
key = sys.argv[1] if len(sys.argv) > 1 else "openhands_heavy40/mars"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = SIM[key]
traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
res = []
for i in range(reps):
    t0 = time.time()
    try:
        run_device_simulation(traces, spec["engine"]["total_blocks"], spec["engine"]["tool_worker_slots"],
                              log=EventLog(), kv_state={})
        res.append("ok")
    except Exception as e:
        res.append("FAIL")
print(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "default"), os.environ.get("MARS_PACK_CTAS", "-"), res)
