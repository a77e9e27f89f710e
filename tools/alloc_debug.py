"""Debug helper: list device allocations per solve (PUMP_DEBUG_ALLOC=1 python tools/alloc_debug.py).
A steady-state solve should allocate nothing."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1607_06886_b200 import api
text = open("scenarios/quad3d_indoor.json").read()
ctx = api.Context(0); sc = api.parse_scenario(text)
for i in range(5):
    print("---- solve", i, file=sys.stderr, flush=True)
    api.run_pump(sc, ctx=ctx)
for i in range(3):
    print("---- e2e solve", i, file=sys.stderr, flush=True)
    api.run_pump(api.parse_scenario(text), ctx=ctx)
