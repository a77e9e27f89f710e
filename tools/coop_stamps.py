"""Per-phase timestamps of the cooperative explore round (PUMP_DEBUG_COOP=1 prints them to stderr).

    PUMP_DEBUG_COOP=1 python tools/coop_stamps.py quad3d_indoor
    PUMP_DEBUG_COOP=1 python tools/coop_stamps.py forest30_n4000
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scenarios"))
import make_scenarios  # noqa: E402
from paper_1607_06886_b200 import api  # noqa: E402

name = sys.argv[1]
if name.startswith("forest30_n"):
    scn = make_scenarios.forest(n_boxes=30)
    scn.update({"samples": int(name[len("forest30_n"):]), "particles": 64, "bank_horizon": 1024})
    text = json.dumps(scn)
else:
    text = open(os.path.join(ROOT, "scenarios", name + ".json")).read()
ctx = api.Context(0)
sc = api.parse_scenario(text)
api.run_pump(sc, ctx=ctx)
print("---- second solve", file=sys.stderr, flush=True)
r = api.run_pump(sc, ctx=ctx)
print("rounds/plans", r["partial_plans"], r["explore_seconds"])
