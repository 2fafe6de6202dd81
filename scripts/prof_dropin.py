"""Host-side profile of the drop-in inside the reference's run_simulation
(demo64/mars, argv[1] to pick another frozen trace): cProfile of the whole
run with GpuMarsPolicy + the B200 balance_and_admit, top functions by own time."""
import cProfile
import json
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(1, os.path.join(ROOT, "baseline", "_ref"))
from agentsched import control, sim, workload  # noqa: E402

from paper_2604_26963_b200.admission import balance_and_admit as gpu_bna  # noqa: E402
from paper_2604_26963_b200.policy import GpuMarsPolicy  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "demo64/mars"
SIM = json.load(open(os.path.join(ROOT, "tests", "golden", "sim_logs.json")))
spec = SIM[key]
traces = workload.load_trace(os.path.join(ROOT, "tests", "golden", spec["trace"]))
params = sim.EngineParams(**spec["engine"])
run = dict(spec["run"])
if "controller" in run:
    run["controller"] = control.ControllerConfig(**run["controller"])
sim.balance_and_admit = gpu_bna
for it in range(2):
    pol = GpuMarsPolicy()
    pol._engine()
    prof = cProfile.Profile()
    t0 = time.perf_counter()
    if it:
        prof.enable()
    res = sim.run_simulation(traces, params, pol, **run)
    if it:
        prof.disable()
    print("wall", time.perf_counter() - t0, "events", len(res.events))
    pol.close()
st = pstats.Stats(prof)
st.sort_stats("tottime").print_stats(30)
