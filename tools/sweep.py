"""Scenario and scaling sweep on one GPU (BASELINE configs[0], [2] and [4]).

    python tools/sweep.py named 3 oracle > gpurun_out/sweep_named.jsonl  # the named scenarios, + oracle check
    python tools/sweep.py scaling 3 oracle > gpurun_out/sweep_scaling.jsonl  # samples x particles x obstacles,
        one axis at a time, oracle parity on the ORACLE_POINTS (the host oracle finishes them in seconds)

One JSON line per workload: ms per solve (CUDA events on the library stream,
L2 flushed before each solve, median of K), the reference's phase split
(pump.hpp:182-261), partial plans, edges, and the per-family kernel times of
one profiled solve.  Variants are derived from the named scenarios' JSON
(scenarios/make_scenarios.py): `samples`, `particles`, and the forest
generator's box count (obstacle sweep in the 40 x 40 x 8 m forest world).
"""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scenarios"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import make_scenarios  # noqa: E402
from paper_1607_06886_b200 import api  # noqa: E402


def named(name):
    with open(os.path.join(ROOT, "scenarios", name + ".json")) as f:
        return json.load(f)


def variants(kind):
    if kind == "named":
        for n in ("quad3d_three_obstacle", "quad3d_indoor", "quad3d_forest"):
            yield n, named(n)
        return
    # scaling (configs[4]): one axis at a time, on worlds that explore
    # (> 1e5 partial plans): samples and particles around quad3d_indoor,
    # obstacles in the quad3d_forest world (40 x 40 x 8 m, n = 16000, N = 128)
    base = named("quad3d_indoor")
    for n in (2000, 4000, 8000, 16000, 32000, 64000):
        yield f"indoor_n{n}_N64", dict(base, samples=n)
    for p in (16, 32, 128, 256):
        yield f"indoor_n4000_N{p}", dict(base, particles=p)
    fb = named("quad3d_forest")
    for k in (3, 10, 30, 100, 300, 1000):
        s = make_scenarios.forest(n_boxes=k)
        s.update({key: fb[key] for key in ("samples", "particles", "alpha", "bank_horizon", "mc_samples",
                                           "connection_radius") if key in fb})
        yield f"forest{k}_n16000_N128", s


ORACLE_POINTS = {"quad3d_three_obstacle", "quad3d_indoor", "quad3d_forest", "indoor_n2000_N64", "indoor_n4000_N64",
                 "indoor_n4000_N16", "indoor_n4000_N32", "indoor_n8000_N64", "indoor_n4000_N128",
                 "indoor_n4000_N256", "forest3_n16000_N128", "forest10_n16000_N128", "forest30_n16000_N128",
                 "forest100_n16000_N128", "forest300_n16000_N128"}


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "named"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    check = len(sys.argv) > 3 and sys.argv[3] == "oracle"  # also solve on the host oracle and compare
    L = api.lib()
    L.pump_ctx_profile.argtypes = [C.c_void_p, C.c_int]
    L.pump_ctx_profile_read.argtypes = [C.c_void_p] * 4
    L.pump_ctx_flush_l2.argtypes = [C.c_void_p]
    L.pump_ctx_stream.argtypes = [C.c_void_p, C.c_void_p]
    ctx = api.Context(0)
    sp = C.c_void_p()
    L.pump_ctx_stream(ctx.h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
    for name, scn in variants(kind):
        line = {"workload": name, "samples": scn["samples"], "particles": scn["particles"],
                "obstacles": len(scn["workspace"]["obstacles"]), "alpha": scn["alpha"]}
        try:
            sc = api.parse_scenario(json.dumps(scn))
            r = api.run_pump(sc, ctx=ctx)  # warm-up (buffers sized)
            ms = []
            for _ in range(reps):
                L.pump_ctx_flush_l2(ctx.h)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = api.run_pump(sc, ctx=ctx)
                e1.record(stream)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            L.pump_ctx_profile(ctx.h, 1)
            L.pump_ctx_flush_l2(ctx.h)
            rp = api.run_pump(sc, ctx=ctx)
            fam = len(bench.FAMILIES)
            pm, pn, pw = np.zeros(fam), np.zeros(fam, dtype=np.int64), np.zeros(fam, dtype=np.int64)
            L.pump_ctx_profile_read(ctx.h, pm.ctypes.data_as(C.c_void_p), pn.ctypes.data_as(C.c_void_p),
                                    pw.ctypes.data_as(C.c_void_p))
            L.pump_ctx_profile(ctx.h, 0)
            # per-family roofline fractions (bench.py's work models)
            peak = C.c_double()
            L.pump_peak_fp64.argtypes = [C.c_void_p, C.c_void_p]
            L.pump_peak_fp64(ctx.h, C.byref(peak))
            dw = len(scn["workspace"]["bounds"]["lo"])
            d = 2 * dw
            F = bench.FAMILIES
            roof = {}
            for f, ops in (("regions", 1.0), ("expand", 2.0 * dw), ("mc_table", bench.mc_table_ops_per_step(d, dw))):
                i = F.index(f)
                if pn[i] > 0 and pm[i] > 0:
                    roof[f] = {"fp64_frac": round(pw[i] * ops / (pm[i] * 1e-3) / 1e9 / peak.value, 4),
                               "ms": round(float(pm[i]), 3)}
            i = F.index("expand")
            if pm[i] > 0:
                Wm = (scn["particles"] + 63) // 64
                hb = rp["partial_plans"] * (2 * 8 * Wm + 32) + rp["explore_hs_read"] * (dw + 1) * 8
                roof["expand"]["hbm_frac"] = round(hb / (pm[i] * 1e-3) / 1e9 / 6553.3, 4)
            line.update({
                "ms_per_solve": round(statistics.median(ms), 3), "reps": reps, "roofline": roof,
                "build_graph_ms": round(1e3 * r["build_graph_seconds"], 3),
                "explore_ms": round(1e3 * r["explore_seconds"], 3),
                "selection_ms": round(1e3 * r["selection_seconds"], 3),
                "success": r["success"], "cost": r["cost"], "certified_cp": r["certified_cp"],
                "partial_plans": r["partial_plans"], "n_edges": r["n_edges"],
                "partial_plans_per_s": round(r["partial_plans"] / r["explore_seconds"], 1)
                if r["explore_seconds"] > 0 else None,
                "kernels_ms": {bench.FAMILIES[i]: round(float(pm[i]), 3) for i in range(fam) if pn[i] > 0}})
            if check and (kind == "named" or name in ORACLE_POINTS):
                import time

                import oracle

                t0 = time.perf_counter()
                o = oracle.run_pump(json.dumps(scn), workers=os.cpu_count() or 1)
                bits = lambda a: np.ascontiguousarray(a).view(np.uint64).tolist()  # noqa: E731
                line["oracle"] = {"ms": round(1e3 * (time.perf_counter() - t0), 1), "cores": os.cpu_count(),
                                  "identical_result": bool(o["path"].tolist() == r["path"].tolist()
                                                           and o["cost"] == r["cost"]
                                                           and o["certified_cp"] == r["certified_cp"]
                                                           and o["partial_plans"] == r["partial_plans"]
                                                           and bits(o["pareto_cp"]) == bits(r["pareto_cp"])
                                                           and bits(o["pareto_cost"]) == bits(r["pareto_cost"])
                                                           and o["mc_eval_ids"].tolist() == r["mc_eval_ids"].tolist()
                                                           and bits(o["traj_pos"]) == bits(r["traj_pos"]))}
            del sc
        except Exception as e:  # report and continue with the next workload
            line["error"] = f"{type(e).__name__}: {e}"
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
