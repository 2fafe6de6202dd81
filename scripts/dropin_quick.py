"""The drop-in's steps/s inside the reference's run_simulation (bench.py's
dropin_sweep / dropin_scale), without the rest of the bench."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for r in bench.dropin_sweep():
    print(json.dumps({"trace": r["trace"], "ref": round(r["reference"]["steps_per_s"]),
                      "b200": round(r["b200"]["steps_per_s"]),
                      "identical": r["b200"]["log_identical"]}))
for r in bench.dropin_scale():
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
