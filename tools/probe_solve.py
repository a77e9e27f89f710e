"""Quick phase timing of one solve (GPU) and the CPU oracle on the same box."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_06886_b200 import api
import oracle

name = sys.argv[1] if len(sys.argv) > 1 else "quad3d_indoor"
cpu = "--cpu" in sys.argv
txt = open(os.path.join("scenarios", name + ".json")).read()
ctx = api.Context(0)
sc = api.parse_scenario(txt)
for it in range(3):
    t = time.perf_counter()
    r = api.run_pump(sc, ctx=ctx)
    dt = time.perf_counter() - t
    keys = ["success", "cost", "certified_cp", "partial_plans", "n_edges", "n_plans", "build_graph_seconds",
            "explore_seconds", "selection_seconds", "bank_ms", "explore_kernel_ms", "mc_ms", "mc_rollouts", "n_mc_evals"]
    print(f"GPU solve {dt*1e3:.1f} ms", {k: r[k] for k in keys}, "launches", ctx.launches, flush=True)
if cpu:
    t = time.perf_counter()
    o = oracle.run_pump(txt, workers=os.cpu_count())
    dt = time.perf_counter() - t
    print(f"CPU oracle solve {dt:.2f} s on {os.cpu_count()} threads", {k: o[k] for k in ["success", "cost", "certified_cp", "partial_plans", "build_graph_seconds", "explore_seconds", "selection_seconds"]})
    same = list(o["path"]) == list(r["path"]) and o["certified_cp"] == r["certified_cp"] and o["cost"] == r["cost"]
    print("identical:", same)
