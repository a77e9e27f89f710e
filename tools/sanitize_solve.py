"""One small solve for compute-sanitizer (tools/sanitize.sh): the scenario
file, with an optional sample / MC cap so memcheck / racecheck finish."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_06886_b200 import api  # noqa: E402

path, samples, mc = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
j = json.load(open(path))
if samples > 0:
    j["samples"] = samples
j["mc_samples"] = mc
ctx = api.Context(0)
r = api.run_pump(api.parse_scenario(json.dumps(j)), ctx=ctx)
print("solve ok", r["success"], r["partial_plans"], r["certified_cp"])
