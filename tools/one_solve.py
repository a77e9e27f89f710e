"""One warm-up solve + one solve (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_06886_b200 import api
name = sys.argv[1] if len(sys.argv) > 1 else "quad3d_indoor"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = api.Context(0)
sc = api.parse_scenario(open(os.path.join("scenarios", name + ".json")).read())
for _ in range(reps):
    r = api.run_pump(sc, ctx=ctx)
print("ok", r["success"], r["partial_plans"], ctx.launches)
