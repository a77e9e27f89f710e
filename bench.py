"""PUMP solve benchmark (BASELINE.json metric) on B200.

Default workload = the largest single-GPU BASELINE config, configs[2]: the
cluttered forest quadrotor scenario (scenarios/quad3d_forest.json: 6-D double
integrator, 200 synthetic AABBs, n = 16000 samples, 128 particles per plan,
alpha = 5%, bisection + MC certification with 20000 rollouts, > 1e5 partial
plans).  One step = one full PUMP solve (pump.hpp:170-263): Halton sampling,
graph build, particle bank, Pareto exploration, Alg. 4 bisection with MC
certification and CP-constrained smoothing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config quad3d_forest|quad3d_indoor|quad3d_three_obstacle] [--no-cpu-baseline]

Prints one JSON line on rank 0.  `value` = ms per solve with the scenario
already parsed (the solve is a synchronous library call whose hot loops all
run on the GPU; the host only orchestrates); `e2e` = the same solve through
the C ABI starting from the JSON scenario text on the host and ending with the
result arrays on the host.  Per-kernel times come from CUDA events recorded
on the library stream around every launch of a second timed pass.  Under
torchrun (N > 1) every rank runs the solve with the MC certification rollouts
and the graph rows sharded across ranks (NCCL all-reduce of the int64 hit
counts, grouped broadcasts of the row slices); time is the max over ranks.

--impl reference times the reference's own CPU code (oracle/_ref: the
reference headers compiled in place, glibc normals) on all host threads, one
bounded sample of the solve per step (see ref_arm below); the oracle
restatement stands in only when oracle/_ref was not built.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FAMILIES = ["bank_noise", "bank_rec", "hsmc", "mc", "connect", "collide", "emit", "regions", "expand", "round_tail",
            "dom", "scan", "multisplit", "misc", "pair_filter", "mc_table"]
SIDE_FAMILIES = ("bank_noise", "bank_rec", "mc_table")  # side stream (capi_plan.cu: c.side)


def mc_table_ops_per_step(d: int, dw: int) -> float:
    """Algorithmic FP64 arithmetic per rollout-step of the MC table build
    (compares excluded), counting only the non-zero terms of the
    axis-separable closed loop the kernels evaluate: (d + dw) normals x 92 ops
    (2 unit maps, log 28, cos 56 by the definition form, sqrt, scaling); per
    axis the 2x2 Sv, 1x1 Sw, 4x2 Gv, 4x1 Gw, 4x4 F blocks, the state sum and
    the output map (79 ops)."""
    return (d + dw) * 92 + 79 * dw


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for k, nm in enumerate(names):
                if s[4 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_text(config: str) -> str:
    with open(os.path.join(ROOT, "scenarios", config + ".json")) as f:
        return f.read()


def config_of(name: str, scn: dict) -> dict:
    """The workload description both arms print (identical dicts)."""
    return {"workload": name, "samples": scn["samples"], "particles": scn["particles"], "alpha": scn["alpha"],
            "mc_samples": scn["mc_samples"], "obstacles": len(scn["workspace"]["obstacles"]),
            "l2": "256 MiB buffer overwritten before every timed solve (GPU arm)"}


ROW_STRIDE, MC_STRIDE = 8, 8  # reference-arm sample: 1/8 of the graph rows, 1/8 of each certification's rollouts


class RefArm:
    """The reference's own code on the host (oracle/_ref/libpumpref.so: the
    unmodified reference headers compiled in place by oracle/ref/Makefile).

    A full forest solve takes tens of seconds on the host, so a step is a
    bounded sample of it (oracle/ref/ref_driver.cpp ref_bench_*): setup builds
    the graph and runs one complete solve (timed: `full_solve_ms`, and its MC
    calls recorded); each step re-runs sample_free, the build_graph row loop
    over every ROW_STRIDE-th source row (x ROW_STRIDE), presample_bank +
    explore on the full graph, and every recorded mc_certify call over its
    first n_mc / MC_STRIDE rollouts (x MC_STRIDE)."""

    def __init__(self, text: str, workers: int):
        import ctypes as C

        import numpy as np

        path = os.path.join(ROOT, "oracle", "_ref", "libpumpref.so")
        self.L = C.CDLL(path)
        self.L.ref_last_error.restype = C.c_char_p
        self.L.ref_bench_setup.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p]
        self.L.ref_bench_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        self.L.ref_bench_free.argtypes = [C.c_void_p]
        self.C, self.np = C, np
        out = np.zeros(9)
        self.h = C.c_void_p()
        if self.L.ref_bench_setup(text.encode(), workers, out.ctypes.data_as(C.c_void_p), C.byref(self.h)) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        self.full_ms = 1e3 * (out[0] + out[1])
        self.setup = {"build_graph_ms": round(1e3 * out[0], 1), "explore_ms": round(1e3 * out[2], 1),
                      "selection_ms": round(1e3 * out[3], 1), "partial_plans": int(out[4]),
                      "mc_calls": int(out[5]), "success": int(out[6]), "cost": float(out[7]), "nodes": int(out[8])}

    def step(self, workers: int, k: int, row_stride: int = ROW_STRIDE, mc_stride: int = MC_STRIDE) -> dict:
        out = self.np.zeros(9)
        if self.L.ref_bench_step(self.h, workers, row_stride, k % row_stride, mc_stride,
                                 out.ctypes.data_as(self.C.c_void_p)) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        return {"est_ms": 1e3 * out[8], "sample_ms": 1e3 * (out[0] + out[1] + out[2] + out[3]),
                "rows": int(out[4]), "partial_plans": int(out[6])}

    def close(self):
        self.L.ref_bench_free(self.h)


def have_ref() -> bool:
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libpumpref.so"))


def run_reference(args, world, rank):
    """The reference's CPU path on the host cores, same config / metric /
    steps / warm-up as the GPU arm.  Rank 0 only."""
    if rank != 0:
        return
    text = load_text(args.config)
    scn = json.loads(text)
    cores = os.cpu_count() or 1
    line = {"impl": "reference", "metric": "PUMP solve time", "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (Halton samples of the named scenario, counter-hash particles/rollouts)",
            "config": config_of(args.config, scn)}
    if have_ref():
        arm = RefArm(text, cores)
        for k in range(args.warmup):
            arm.step(cores, k)
        times, samples = [], []
        for k in range(args.steps):
            r = arm.step(cores, args.warmup + k)
            times.append(r["est_ms"])
            samples.append(r["sample_ms"])
        arm.close()
        ms = sum(times) / len(times)
        line.update({"value": round(ms, 3), "ms_per_step": round(ms, 3),
                     "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": cores, "kind": "reference",
                                      "sample": f"per step: sample_free + build_graph rows v = k (mod {ROW_STRIDE}) "
                                                f"(x{ROW_STRIDE}) + presample_bank + explore (full) + the solve's "
                                                f"mc_certify calls on 1/{MC_STRIDE} of their rollouts "
                                                f"(x{MC_STRIDE}); oracle/_ref, workers = all host threads",
                                      "sample_ms_per_step": round(sum(samples) / len(samples), 1),
                                      "full_solve_ms": round(arm.full_ms, 1), "full_solve": arm.setup},
                     "partial_plans": arm.setup["partial_plans"], "success": arm.setup["success"]})
    else:  # oracle/_ref not built: the oracle restatement, full solves
        import oracle

        for _ in range(min(args.warmup, 1)):
            oracle.run_pump(text, workers=cores)
        times, r = [], None
        for _ in range(args.steps):
            t0 = time.perf_counter()
            r = oracle.run_pump(text, workers=cores)
            times.append(time.perf_counter() - t0)
        ms = 1e3 * sum(times) / len(times)
        line.update({"value": round(ms, 3), "ms_per_step": round(ms, 3),
                     "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": cores, "kind": "port",
                                      "sample": "one full solve per step (oracle restatement, all host threads)"},
                     "partial_plans": r["partial_plans"], "success": r["success"]})
    line["e2e"] = {"value": line["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="quad3d_forest")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mc-sweep", action="store_true")
    ap.add_argument("--no-rrt", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # >= 3 warm-up steps (both arms)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import numpy as np

    from paper_1607_06886_b200 import api
    import ctypes as C

    L = api.lib()
    L.pump_ctx_profile.argtypes = [C.c_void_p, C.c_int]
    L.pump_ctx_profile_read.argtypes = [C.c_void_p] * 4
    L.pump_ctx_io_bytes.argtypes = [C.c_void_p, C.c_void_p]
    L.pump_ctx_flush_l2.argtypes = [C.c_void_p]
    L.pump_peak_fp64.argtypes = [C.c_void_p, C.c_void_p]
    L.pump_probe_round_latency.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]

    text = load_text(args.config)
    scn = json.loads(text)
    ctx = api.Context(local)
    sc = api.parse_scenario(text)
    if world > 1 and hasattr(api, "set_comm"):
        api.set_comm(ctx, rank, world)

    def io():
        b = np.zeros(5, dtype=np.int64)
        L.pump_ctx_io_bytes(ctx.h, b.ctypes.data_as(C.c_void_p))
        return b

    # warm-up (buffers sized, modules loaded)
    res = None
    for _ in range(args.warmup):
        res = api.run_pump(sc, ctx=ctx)

    # ---- timed region: K solves timed with CUDA events on the library's own
    # stream (every kernel and copy of a solve is ordered on it), L2 flushed
    # before each; the per-kernel profiler is OFF here (its per-launch events
    # would inflate the step)
    import torch

    L.pump_ctx_stream.argtypes = [C.c_void_p, C.c_void_p]
    sp = C.c_void_p()
    L.pump_ctx_stream(ctx.h, C.byref(sp))
    lib_stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", local))
    L.pump_ctx_flush_l2(ctx.h)  # allocate the flush buffer outside the timed region

    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launches
    io0 = io()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for k in range(args.steps):
        L.pump_ctx_flush_l2(ctx.h)  # synchronous: the stream is idle when the start event is recorded
        evs[k][0].record(lib_stream)
        res = api.run_pump(sc, ctx=ctx)  # returns after the result is on the host
        evs[k][1].record(lib_stream)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    io1 = io()
    launches = ctx.launches - launches0
    clk = clocks.stop()
    barrier(world)
    ms_per_step = max_over_ranks(sum(step_ms) / len(step_ms), world)

    # ---- profiled pass (same workload, K more solves): per-launch CUDA events
    # on the library stream, per kernel family -> "kernels" and "roofline"
    L.pump_ctx_profile(ctx.h, 1)
    res_prof = None
    for _ in range(args.steps):
        L.pump_ctx_flush_l2(ctx.h)
        res_prof = api.run_pump(sc, ctx=ctx)  # (work counters such as the expand half-space count run here)
    prof_ms = np.zeros(len(FAMILIES))
    prof_n = np.zeros(len(FAMILIES), dtype=np.int64)
    prof_w = np.zeros(len(FAMILIES), dtype=np.int64)
    L.pump_ctx_profile_read(ctx.h, prof_ms.ctypes.data_as(C.c_void_p), prof_n.ctypes.data_as(C.c_void_p),
                            prof_w.ctypes.data_as(C.c_void_p))
    L.pump_ctx_profile(ctx.h, 0)

    # ---- e2e: JSON text on the host -> parse -> solve -> result arrays on the host
    barrier(world)
    e_io0 = io()
    e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        L.pump_ctx_flush_l2(ctx.h)
        e_evs[k][0].record(lib_stream)  # GPU timestamps: host parse time (stream idle) is inside the span
        s2 = api.parse_scenario(text)
        r2 = api.run_pump(s2, ctx=ctx)
        e_evs[k][1].record(lib_stream)
        del s2
    torch.cuda.synchronize()
    e_ms = [a.elapsed_time(b) for a, b in e_evs]
    e_io1 = io()
    e2e_ms = max_over_ranks(sum(e_ms) / len(e_ms), world)
    assert r2["path"].tolist() == res["path"].tolist() and r2["certified_cp"] == res["certified_cp"]

    # ---- the same solve with a prebuilt graph (run_pump's `prebuilt`,
    # pump.hpp:170-171; SURVEY §8d asks for both): the graph is built once from
    # the scenario's own node set outside the timed solves
    prm = sc.params()
    pos, vel = sc.nodes()
    g_pre = api.build_graph(pos, vel, sc.workspace(), sc.goal(), prm["r_n"], prm["dt"], prm["eps_cc"],
                            prm["tau_max"], ctx=ctx)
    for _ in range(2):
        api.run_pump(sc, prebuilt=g_pre, ctx=ctx)
    p_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        L.pump_ctx_flush_l2(ctx.h)
        p_evs[k][0].record(lib_stream)
        r3 = api.run_pump(sc, prebuilt=g_pre, ctx=ctx)
        p_evs[k][1].record(lib_stream)
    torch.cuda.synchronize()
    pre_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in p_evs) / args.steps, world)
    assert r3["path"].tolist() == res["path"].tolist() and r3["certified_cp"] == res["certified_cp"]
    del g_pre

    # ---- the Table 1 baseline on the same scenario: repeated RRT (rrt.hpp,
    # the scenario's trials / alpha / mc_samples), trials and certification on the GPU
    rrt = None
    if not args.no_rrt:
        api.repeated_rrt(sc, ctx=ctx)  # warm-up (buffers)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(lib_stream)
        rr = api.repeated_rrt(sc, ctx=ctx)
        e1.record(lib_stream)
        torch.cuda.synchronize()
        rrt = {"ms": round(max_over_ranks(e0.elapsed_time(e1), world), 3), "success": rr["success"],
               "cost": rr["cost"], "certified_cp": rr["certified_cp"],
               "trials": int(scn.get("rrt", {}).get("trials", 1000)),
               "trials_reaching_goal": rr["trials_reaching_goal"],
               "certification_attempts": rr["certification_attempts"],
               "pump_cost_le_rrt_cost": bool(res["success"] and (not rr["success"] or res["cost"] <= rr["cost"] + 1e-9))}

    # ---- MC certification sweep: mc_certify of the
    # certified trajectory with n_mc in {1e4 .. 1e7}, rollouts sharded over
    # the ranks ([n r / W, n (r+1) / W)), hit counts summed across ranks
    sweep = []
    if not args.no_mc_sweep:
        cl, wsd = sc.closed_loop(), sc.workspace()
        traj = np.ascontiguousarray(res["traj_pos"])
        for n_mc in (10 ** 4, 10 ** 5, 10 ** 6, 10 ** 7):
            lo, hi = api.shard_range(n_mc, rank, world)
            api.mc_certify_batch(cl, wsd, [traj], lo, hi, prm["seed_mc"], prm["eps_cc"], ctx)  # warm-up (buffers)
            barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(lib_stream)
            hits = api.mc_certify_batch(cl, wsd, [traj], lo, hi, prm["seed_mc"], prm["eps_cc"], ctx)
            e1.record(lib_stream)
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1), world)
            total = int(hits[0])
            if world > 1:
                import torch.distributed as dist

                t = torch.tensor([total], dtype=torch.int64, device="cuda")
                dist.all_reduce(t)
                total = int(t.item())
            sweep.append({"n_mc": n_mc, "ms": round(ms, 3), "rollouts_per_s": round(n_mc / (ms * 1e-3), 1),
                          "rollout_steps_per_s": round(n_mc * len(traj) / (ms * 1e-3), 1),
                          "cp": total / n_mc})

    # ---- roofline of the dominant kernel family (CUDA events, profiled pass),
    # plus the same figures for every family with a work model
    peak = C.c_double()
    L.pump_peak_fp64(ctx.h, C.byref(peak))
    us_bar, us_l2 = C.c_double(), C.c_double()
    L.pump_probe_round_latency(ctx.h, C.byref(us_bar), C.byref(us_l2))
    hbm = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm = None
    d, dw = 2 * len(scn["workspace"]["bounds"]["lo"]), len(scn["workspace"]["bounds"]["lo"])
    n_obs = len(scn["workspace"]["obstacles"])

    ROUND_TAIL_BARRIERS = 10  # grid_sync() calls in k_round_tail (explore.cu)

    def roofline_of(fam):
        name = FAMILIES[fam]
        r = {"kernel": name, "bound": "fp64", "unit": "GFLOP/s", "peak": round(peak.value, 1),
             "peak_source": "measured: bench FP64 DMUL+DADD issue microbenchmark (no FMA, the parity op mix); "
                            "MEASURED_PEAKS.json has no FP64 figure",
             "share_of_step": round(float(prof_ms[fam] / max(1e-9, prof_ms.sum())), 3),
             "avg_launch_ms": round(float(prof_ms[fam] / max(1, prof_n[fam])), 4), "launches": int(prof_n[fam]),
             "traffic": None}
        t = prof_ms[fam] * 1e-3
        if name == "mc_table":
            opw = mc_table_ops_per_step(d, dw)
            work = prof_w[fam] * opw
            r["work"] = f"{int(prof_w[fam])} rollout-steps drawn x {opw:.0f} FP64 ops"
        elif name == "expand":
            work = prof_w[fam] * 2 * dw
            r["work"] = f"{int(prof_w[fam])} particle-halfspace tests performed x {2 * dw} FP64 ops"
            # SURVEY §8d K_hsmc HBM-byte model: per task the parent mask in and
            # the candidate mask out (8 W bytes each), the 32-byte record, and
            # every half-space of the edge's waypoints ((dw + 1) x 8 bytes)
            Wm = (scn["particles"] + 63) // 64
            hbm_bytes = res_prof["partial_plans"] * (2 * 8 * Wm + 32) + res_prof["explore_hs_read"] * (dw + 1) * 8
            t_solve = prof_ms[fam] / args.steps * 1e-3
            r["hbm_model"] = {"bytes_per_solve": int(hbm_bytes),
                              "achieved_gbs": round(hbm_bytes / t_solve / 1e9, 1) if t_solve > 0 else None,
                              "peak_gbs": hbm, "frac": round(hbm_bytes / t_solve / 1e9 / hbm, 5)
                              if (t_solve > 0 and hbm) else None,
                              "model": "tasks x (2 x 8 W mask + 32 record) + half-spaces read x (dw + 1) x 8"}
        elif name == "regions":
            work = prof_w[fam]
            r["work"] = (f"{int(prof_w[fam])} FP64-pipe ops of the region loop (14 per box distance, 10 per prune "
                         "test, counted in the kernel)")
        elif name == "round_tail":
            r.update({"bound": "hbm", "unit": "GB/s", "peak": hbm,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"})
            work = prof_w[fam]
            r["work"] = f"{int(prof_w[fam])} algorithmic bytes (candidate records, arena writes, pool, group)"
            # the bound that actually binds: the dependent grid-barrier chain
            # (ROUND_TAIL_BARRIERS grid syncs per launch, each measured live
            # on the round kernel's own grid shape)
            avg_us = 1e3 * float(prof_ms[fam] / max(1, prof_n[fam]))
            floor_us = ROUND_TAIL_BARRIERS * us_bar.value
            r["latency_floor"] = {"barriers_per_launch": ROUND_TAIL_BARRIERS,
                                  "us_per_grid_barrier": round(us_bar.value, 3),
                                  "us_per_dependent_l2_load": round(us_l2.value, 4),
                                  "floor_us_per_launch": round(floor_us, 2), "avg_launch_us": round(avg_us, 2),
                                  "frac": round(floor_us / avg_us, 3) if avg_us > 0 else None}
        else:
            r["work"] = None
            r["achieved"] = None
            r["frac"] = None
            return r
        achieved = work / t / 1e9 if t > 0 else 0.0
        r["achieved"] = round(achieved, 1)
        r["frac"] = round(achieved / r["peak"], 5) if r.get("peak") else None
        return r

    # ncu DRAM traffic per launch of the family's kernel (committed --set full
    # captures, tools/ncu_kernels.py; cold-cache, one launch each)
    ncu_rows = []
    for f in ("r2_ncu_kernels.json", "r1_ncu_kernels.json"):
        try:
            with open(os.path.join(ROOT, "profiles", f)) as fh:
                ncu_rows = [dict(d, source=f) for d in json.load(fh)["kernels"]]
            break
        except Exception:
            continue
    FAM_KERNEL = {"regions": "k_regions_once", "round_tail": "k_round_tail", "expand": "k_expand",
                  "pair_filter": "k_pair_filter_grid", "bank_rec": "k_bank_rec_sep", "mc_table": "k_mcnoise_sep",
                  "connect": "k_connect", "collide": "k_collide", "mc": "k_mc_tab"}

    def with_traffic(r):
        pre = FAM_KERNEL.get(r["kernel"])
        for d in ncu_rows:
            if pre and d["kernel"].startswith(pre):
                r["traffic"] = int(d.get("dram_read", 0) + d.get("dram_write", 0))
                r["traffic_source"] = f"profiles/{d['source']} ({d['kernel']}, ncu dram__bytes_read + write, one launch)"
                break
        return r

    # the dominant family of the solve's critical path: the largest one on the
    # library stream (the bank and the MC table run on the side stream,
    # overlapped with the graph build and the explore rounds)
    main_ms = np.array([0.0 if FAMILIES[i] in SIDE_FAMILIES else prof_ms[i] for i in range(len(FAMILIES))])
    roof = with_traffic(roofline_of(int(np.argmax(main_ms))))
    roof["selection"] = "largest kernel family on the library stream (side-stream bank / MC-table families excluded)"
    rooflines = [with_traffic(roofline_of(FAMILIES.index(f))) for f in ("regions", "expand", "round_tail", "mc_table")
                 if prof_n[FAMILIES.index(f)] > 0]
    kernels = {FAMILIES[i]: {"ms_per_step": round(float(prof_ms[i] / args.steps), 3),
                             "launches_per_step": round(float(prof_n[i] / args.steps), 1)}
               for i in range(len(FAMILIES)) if prof_n[i] > 0}

    # ---- CPU baseline: the reference path (oracle restatement) on this host
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        o = oracle.run_pump(text, workers=cores)
        cpu_s = time.perf_counter() - t0
        bits = lambda a: np.ascontiguousarray(a).view(np.uint64).tolist()  # noqa: E731
        same = (o["path"].tolist() == res["path"].tolist() and o["certified_cp"] == res["certified_cp"]
                and o["cost"] == res["cost"] and o["partial_plans"] == res["partial_plans"]
                and bits(o["pareto_cost"]) == bits(res["pareto_cost"]) and bits(o["pareto_cp"]) == bits(res["pareto_cp"])
                and o["mc_eval_ids"].tolist() == res["mc_eval_ids"].tolist()
                and bits(o["mc_eval_values"]) == bits(res["mc_eval_values"])
                and bits(o["traj_pos"]) == bits(res["traj_pos"]) and o["smoothing_s"] == res["smoothing_s"])
        cpu = {"value": round(1e3 * cpu_s, 1), "unit": "ms", "cores": cores, "kind": "port",
               "sample": "one full solve of the same scenario (oracle restatement, workers = all host threads)",
               "identical_result": bool(same),
               "compared": "path, cost, certified CP, partial plans, Pareto front (cost, cp bits), MC probe ids and "
                           "values, smoothing fraction, trajectory position bits"}
        if have_ref():
            # the reference's own code (oracle/_ref): one full solve on all
            # threads, and a bounded 1-thread sample (the same RefArm steps
            # with 1/64 of the rows and of each certification's rollouts)
            arm = RefArm(text, cores)
            one = arm.step(1, 0, 64, 64)
            cpu["reference"] = {"kind": "reference", "cores": cores, "full_solve_ms": round(arm.full_ms, 1),
                                "phases": arm.setup}
            cpu["workers_1"] = {"kind": "reference", "cores": 1, "value": round(one["est_ms"], 1), "unit": "ms",
                                "sample": "sample_free + build_graph rows v = 0 (mod 64) (x64) + bank + explore "
                                          "(full) + the solve's mc_certify calls on 1/64 of their rollouts (x64)",
                                "sample_ms": round(one["sample_ms"], 1)}
            arm.close()

    # per-kernel roofline table from the committed ncu --set full captures
    # (tools/ncu_kernels.py; static evidence, not measured in this run)
    ncu_tab = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_kernels.json")) as f:
            nk = json.load(f)
        ncu_tab = {"source": "profiles/r2_ncu_kernels.json (ncu --set full on quad3d_forest, one launch each; "
                             "not this run)",
                   "kernels": [{k: d.get(k) for k in ("kernel", "dur_us", "bound", "frac", "fp64_pipe_pct",
                                                       "issue_pct", "dram_gbs")} for d in nk["kernels"]]}
    except Exception:
        ncu_tab = None

    pp_s = res["partial_plans"] / (res["explore_seconds"]) if res["explore_seconds"] > 0 else None
    # certification rollouts per second of the solve's MC work: the
    # certification kernels plus the common-random-number table they read
    mc_tab_ms = float(prof_ms[FAMILIES.index("mc_table")] / args.steps)
    mc_rs = res["mc_rollouts"] / ((res["mc_ms"] + mc_tab_ms) * 1e-3) if res["mc_ms"] > 0 else None
    line = {
        "metric": "PUMP solve time", "value": round(ms_per_step, 3), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Halton samples of the named scenario; counter-hash particle bank and MC rollouts)",
        "config": config_of(args.config, scn),
        "timing": "CUDA events on the library stream around each solve (profiler off); kernels/roofline "
                  "from a second K-solve pass with per-launch events",
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms",
                "h2d_bytes_per_step": int((e_io1[0] - e_io0[0]) // args.steps),
                "d2h_bytes_per_step": int((e_io1[1] - e_io0[1]) // args.steps)},
        "mc_sweep": sweep,
        "rrt_baseline": rrt,
        "prebuilt_graph": {"value": round(pre_ms, 3), "unit": "ms",
                           "note": "run_pump with a prebuilt graph (graph built once from the scenario's nodes)"},
        "gpu_launches": int(launches // args.steps), "gpu_launches_total": int(launches),
        "device_allocs_timed": int(io1[3] - io0[3] + e_io1[3] - e_io0[3]),
        "clocks": clk, "roofline": roof, "rooflines": rooflines, "ncu_kernels": ncu_tab, "cpu_baseline": cpu,
        "kernels": kernels,
        "solve": {"success": res["success"], "cost": res["cost"], "certified_cp": res["certified_cp"],
                  "partial_plans": res["partial_plans"], "n_edges": res["n_edges"], "n_plans": res["n_plans"],
                  "build_graph_ms": round(1e3 * res["build_graph_seconds"], 3),
                  "explore_ms": round(1e3 * res["explore_seconds"], 3),
                  "selection_ms": round(1e3 * res["selection_seconds"], 3)},
        "partial_plans_per_s": round(pp_s, 1) if pp_s else None,
        "mc_rollouts_per_s": round(mc_rs, 1) if mc_rs else None,
        "mc_rollouts_per_s_note": "solve's certified rollouts / (certification kernels + MC-table build) time",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
