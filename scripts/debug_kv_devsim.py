"""Debug: the devsim block-ID run that fails with step status 4 (r2)."""
import os, sys, json, traceback
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MARS_DEBUG_LAUNCH", "1")
from tests.test_gpu_devsim import SIM, SIM_BASE, GOLDEN, VARIANT_KW
from oracle import tracefile
from paper_2604_26963_b200.devsim import run_device_simulation, EventLog
import paper_2604_26963_b200.devsim as D

key = sys.argv[1] if len(sys.argv) > 1 else "small12/mars"
spec = SIM[key] if key in SIM else SIM_BASE[key]
traces = tracefile.load(os.path.join(GOLDEN, spec["trace"]))
variant = key.split("/")[1]
kw = dict(VARIANT_KW.get(variant, {}))
if key in SIM_BASE:
    kw["policy"] = spec["policy"]
for pe in ("20", "0"):
    os.environ["MARS_PACK_CTAS"] = pe
    log, kv = EventLog(), {}
    try:
        run_device_simulation(traces, spec["engine"]["total_blocks"], spec["engine"]["tool_worker_slots"],
                              enable_control_plane=spec["run"].get("enable_control_plane", True),
                              log=log, kv_state=kv, **kw)
        print("PACK", pe, "ok", kv.get("status"))
    except Exception as e:
        print("PACK", pe, "FAIL", repr(e)[:200], "records", len(log.records))
