"""Median per-phase host-clock times (graph, explore, selection) of warm forest solves with
whichever libpump_gpu.so is in place (A/B: tools/ab_phase.sh).   python tools/phase_ab.py [scenario] [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_1607_06886_b200 import api  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "quad3d_forest"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
if name.startswith("forest") and name[6:].isdigit():  # forestK: config 5's obstacle axis (tools/sweep.py)
    import json
    sys.path.insert(0, "scenarios")
    import make_scenarios  # noqa: E402
    fb = json.load(open("scenarios/quad3d_forest.json"))
    s = make_scenarios.forest(n_boxes=int(name[6:]))
    s.update({k: fb[k] for k in ("samples", "particles", "alpha", "bank_horizon", "mc_samples", "connection_radius")
              if k in fb})
    sc = api.parse_scenario(json.dumps(s))
else:
    sc = api.parse_scenario(open(f"scenarios/{name}.json").read())
ctx = api.Context(0)
for _ in range(5):
    api.run_pump(sc, ctx=ctx)
rows = []
for _ in range(n):
    r = api.run_pump(sc, ctx=ctx)
    rows.append([1e3 * r[k] for k in ("build_graph_seconds", "explore_seconds", "selection_seconds")])
med = np.median(np.array(rows), axis=0)
print(name, "graph %.3f explore %.3f selection %.3f (ms, median of %d)" % (*med, n))
