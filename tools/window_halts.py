import json, sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
from paper_1607_06886_b200 import api
for lam in (0.01, 0.05, 0.5):
    j = json.load(open("scenarios/quad3d_three_obstacle.json")); j.update(samples=500, mc_samples=3000)
    j["lambda"] = lam
    r = api.run_pump(api.parse_scenario(json.dumps(j)))
    print("lambda", lam, "partial", r["partial_plans"], file=sys.stderr, flush=True)
