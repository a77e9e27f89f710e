"""One quad3d_indoor solve through the C ABI (ncu target: small, deterministic).

    ncu --set full -k regex:k_mc_sep -c 2 -o prof python tools/prof_solve.py
    python tools/prof_solve.py quad3d_indoor 5      # five solves in one process
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_06886_b200 import api  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "quad3d_indoor"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "scenarios", name + ".json")) as f:
    text = f.read()
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = api.Context(0)
for _ in range(reps):
    r = api.run_pump(api.parse_scenario(text), ctx=ctx)
print("success", r["success"], "cost", r["cost"], "cp", r["certified_cp"])
