"""The drop-in crossover sizes twice in one process (one-time costs vs per tick)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for rep in range(2):
    for r in bench.dropin_scale(sizes=(64, 512, 4096), ticks=int(sys.argv[1]) if len(sys.argv) > 1 else 40, warm=rep == 0):
        print(rep, json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()}))
