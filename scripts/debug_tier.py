"""Debug: openhands devsim with / without the host tier (status 4 hunt)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MARS_DEBUG_LAUNCH", "1")
from oracle import tracefile
from tests._sim import SIM, VARIANT_KW
from tests.conftest import GOLDEN
from paper_2604_26963_b200.devsim import EventLog, run_device_simulation
key = sys.argv[1] if len(sys.argv) > 1 else "openhands_heavy40/mars"
spec = SIM[key]
traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
for name, kw in [("plain", {}), ("kv", {"kv_state": {}}),
                 ("tier", {"kv_state": {}, "kv_tier": {"block_bytes": 1024}}),
                 ("tier+pattern", {"kv_state": {}, "kv_tier": {"block_bytes": 1024, "pattern": True}})]:
    t0 = time.time()
    try:
        run_device_simulation(traces, spec["engine"]["total_blocks"], spec["engine"]["tool_worker_slots"],
                              log=EventLog(), **kw)
        print(name, "ok", round(time.time() - t0, 2), kw.get("kv_tier"))
    except Exception as e:
        print(name, "FAIL", repr(e)[:200], round(time.time() - t0, 2))
