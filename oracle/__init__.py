"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/liboracle.so``: the CPU restatement of the PUMP
reference hot path (see ``pump_oracle.hpp`` for the header, citations and
pinning).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs may import this module, and only as the checker / the timed CPU
baseline.  The product (``paper_1607_06886_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1607_06886_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_normal.restype = C.c_double
        L.oracle_normal.argtypes = [C.c_uint64] * 4
        L.oracle_uniform.restype = C.c_double
        L.oracle_uniform.argtypes = [C.c_uint64] * 4
        L.oracle_counter_hash.restype = C.c_uint64
        L.oracle_counter_hash.argtypes = [C.c_uint64] * 4
        L.oracle_steer_cost.restype = C.c_double
        L.oracle_halton.restype = C.c_double
        L.oracle_halton.argtypes = [C.c_uint64, C.c_int]
        for name in ("oracle_graph_free", "oracle_explore_free", "oracle_result_free"):
            getattr(L, name).argtypes = [vp]
            getattr(L, name).restype = None
        for name in ("oracle_graph_counts", "oracle_graph_export", "oracle_explore_counts",
                     "oracle_explore_export", "oracle_result_summary"):
            getattr(L, name).argtypes = [vp, vp]
        L.oracle_result_arrays.argtypes = [vp] * 10
        L.oracle_explore.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, vp]
        L.oracle_explore_invariants.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]
        L.oracle_run_pump.argtypes = [C.c_char_p, C.c_int, vp, vp]
        L.oracle_graph_from_view.argtypes = [vp, vp]
        L.oracle_build_graph.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_int, vp]
        L.oracle_presample_bank.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_int, vp]
        L.oracle_mc_hits.argtypes = [vp, vp, C.c_int, vp, C.c_int64, C.c_int64, C.c_uint64, C.c_double,
                                     C.c_int, vp, vp]
        L.oracle_hsmc_extend_batch.argtypes = [C.c_int, C.c_int, C.c_int, vp, C.c_int64, C.c_int, vp, vp, vp,
                                               vp, vp, vp, vp, vp, C.c_int]
        L.oracle_connect.argtypes = [C.c_int, vp, vp, vp, vp, C.c_double, vp, vp, vp]
        L.oracle_steer_cost.argtypes = [C.c_int, vp, vp, vp, vp, C.c_double]
        L.oracle_motion_collides.argtypes = [vp, vp, vp, vp, vp, C.c_double, vp, vp, C.c_double, vp]
        L.oracle_point_free.argtypes = [vp, vp]
        L.oracle_segment_collides.argtypes = [vp, vp, vp]
        L.oracle_local_convex_region.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp, vp]
        L.oracle_scenario_nodes.argtypes = [C.c_char_p, C.c_int, vp, vp, vp]
        L.oracle_scenario_closed_loop.argtypes = [C.c_char_p, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_normals.argtypes = [C.c_uint64, C.c_int64, vp, vp, vp, vp]
        L.oracle_set_normal_mode.argtypes = [C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


EXC = {A.PUMP_E_INVALID_ARGUMENT: ValueError, A.PUMP_E_OUT_OF_RANGE: IndexError}


def _check(rc):
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        exc = EXC.get(rc)
        if exc is not None:
            e = exc(msg)
            e.code = rc
            raise e
        raise OracleError(rc, msg)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ------------------------------------------------------------------ normals
PORTABLE, GLIBC = 0, 1


def set_normal_mode(mode: int):
    lib().oracle_set_normal_mode(int(mode))


def normal(seed, a, b, ch):
    return lib().oracle_normal(seed, a, b, ch)


def uniform(seed, a, b, c):
    return lib().oracle_uniform(seed, a, b, c)


def counter_hash(seed, a, b, c):
    return lib().oracle_counter_hash(seed, a, b, c)


def normals(seed, a, b, ch):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(np.broadcast_to(b, a.shape), dtype=np.uint64)
    ch = np.ascontiguousarray(np.broadcast_to(ch, a.shape), dtype=np.uint64)
    out = np.zeros(a.shape, dtype=np.float64)
    lib().oracle_normals(C.c_uint64(seed), a.size, _p(a), _p(b), _p(ch), _p(out))
    return out


def halton(index, base):
    return lib().oracle_halton(index, base)


def bisect_select(values, alpha):
    """bisect_select (pump.hpp:23-51) over ids 0..n-1 with MC values."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    n = v.size
    plan, mc, ne = C.c_int(), C.c_double(), C.c_int()
    ev = np.zeros(max(1, n), dtype=np.int32)
    L = lib()
    L.oracle_bisect_select.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
    ok = L.oracle_bisect_select(n, _p(v) if n else None, alpha, C.byref(plan), C.byref(mc), _p(ev), C.byref(ne))
    return {"success": bool(ok), "plan_id": plan.value, "mc": mc.value, "evals": ev[:ne.value].tolist()}


def fixed_time_connect(ap, av, bp, bv, tau):
    dw = len(ap)
    arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (ap, av, bp, bv)]
    cost = C.c_double()
    a0, j = np.zeros(dw), np.zeros(dw)
    L = lib()
    L.oracle_fixed_time_connect.argtypes = [C.c_int] + [C.c_void_p] * 4 + [C.c_double] + [C.c_void_p] * 3
    L.oracle_fixed_time_connect.restype = None
    L.oracle_fixed_time_connect(dw, *[_p(x) for x in arr], tau, C.byref(cost), _p(a0), _p(j))
    return {"ok": True, "tau": tau, "cost": cost.value, "acc0": a0, "jerk": j}


def waypoints(ap, av, bp, bv, motion, dt, cap=100000):
    """motion_waypoints (steer.hpp:192-212): (t, pos, vel, control) arrays."""
    dw = len(ap)
    arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (ap, av, bp, bv)]
    t, p, v, u = np.zeros(cap), np.zeros((cap, dw)), np.zeros((cap, dw)), np.zeros((cap, dw))
    L = lib()
    L.oracle_waypoints.argtypes = [C.c_int] + [C.c_void_p] * 4 + [C.c_double, C.c_void_p, C.c_void_p, C.c_double,
                                                                 C.c_int] + [C.c_void_p] * 4
    n = L.oracle_waypoints(dw, *[_p(x) for x in arr], motion["tau"], _p(np.ascontiguousarray(motion["acc0"])),
                           _p(np.ascontiguousarray(motion["jerk"])), dt, cap, _p(t), _p(p), _p(v), _p(u))
    return t[:n], p[:n], v[:n], u[:n]


# ------------------------------------------------------------------ models
def scenario_models(json_text: str):
    """(closed-loop dict, scalars dict) of a scenario via the shared host
    synthesis (models.hpp) — the same matrices the product consumes."""
    L = lib()
    d, dw = C.c_int32(), C.c_int32()
    sc = np.zeros(8)
    _check(L.oracle_scenario_closed_loop(json_text.encode(), C.byref(d), C.byref(dw), None, None, None, None,
                                         None, None, None, _p(sc)))
    d, dw = d.value, dw.value
    m = {"F": np.zeros((2 * d, 2 * d)), "Gv": np.zeros((2 * d, d)), "Gw": np.zeros((2 * d, dw)),
         "Sv": np.zeros((d, d)), "Sw": np.zeros((dw, dw)), "S0": np.zeros((d, d)), "C": np.zeros((dw, d))}
    _check(L.oracle_scenario_closed_loop(json_text.encode(), C.byref(C.c_int32()), C.byref(C.c_int32()),
                                         *[_p(m[k]) for k in ("F", "Gv", "Gw", "Sv", "Sw", "S0", "C")], None))
    m["d"], m["dw"] = d, dw
    keys = ["eps_cc", "r_n", "tau_max", "alpha", "eta", "lambda", "dt", "max_speed"]
    return m, dict(zip(keys, sc.tolist()))


# -------------------------------------------------------------------- bank
def presample_bank(cl: dict, t_max: int, n: int, seed: int, workers: int = 1) -> np.ndarray:
    keep = A.Keep()
    s = A.closed_loop_struct(cl, keep)
    out = np.zeros((t_max + 1, n, cl["dw"]))
    _check(lib().oracle_presample_bank(C.byref(s), t_max, n, C.c_uint64(seed), workers, _p(out)))
    return out


# -------------------------------------------------------------------- hsmc
def hsmc_extend_batch(bank: np.ndarray, masks_in, step_off, step_t, step_hs_off, hs_a, hs_b, workers=1):
    bank = np.ascontiguousarray(bank, dtype=np.float64)
    horizon, n, dw = bank.shape[0] - 1, bank.shape[1], bank.shape[2]
    masks_in = np.ascontiguousarray(masks_in, dtype=np.uint64)
    n_tasks, n_words = masks_in.shape
    step_off = np.ascontiguousarray(step_off, dtype=np.int64)
    step_t = np.ascontiguousarray(step_t, dtype=np.int32)
    step_hs_off = np.ascontiguousarray(step_hs_off, dtype=np.int64)
    hs_a = np.ascontiguousarray(hs_a, dtype=np.float64).reshape(-1)
    hs_b = np.ascontiguousarray(hs_b, dtype=np.float64)
    out = np.zeros_like(masks_in)
    pop = np.zeros(n_tasks, dtype=np.int32)
    _check(lib().oracle_hsmc_extend_batch(n, horizon, dw, _p(bank), n_tasks, n_words, _p(masks_in),
                                          _p(step_off), _p(step_t), _p(step_hs_off), _p(hs_a), _p(hs_b),
                                          _p(out), _p(pop), workers))
    return out, pop


# ---------------------------------------------------------------------- mc
def mc_hits(cl: dict, ws: dict, y_nom, r0: int, r1: int, seed: int, eps_cc: float, workers=1,
            want_flags=False):
    keep = A.Keep()
    cls = A.closed_loop_struct(cl, keep)
    wss = A.workspace_struct(ws, keep)
    y = keep.f64(y_nom).reshape(-1, cl["dw"])
    hits = C.c_int64()
    flags = np.zeros(max(0, r1 - r0), dtype=np.uint8) if want_flags else None
    _check(lib().oracle_mc_hits(C.byref(cls), C.byref(wss), y.shape[0], _p(y), r0, r1, C.c_uint64(seed),
                                eps_cc, workers, C.byref(hits), _p(flags)))
    return (hits.value, flags) if want_flags else hits.value


def mc_certify(cl, ws, y_nom, n_mc, seed, eps_cc, workers=1):
    if n_mc < 1:
        raise ValueError("mc_certify: need at least one rollout")
    return mc_hits(cl, ws, y_nom, 0, n_mc, seed, eps_cc, workers) / n_mc


# ------------------------------------------------------------ steer / geom
def smooth(t, pos, vel, ctrl, plan_mc, alpha, cl, ws, n_mc, seed, eps_cc, workers=1) -> dict:
    """pump.hpp:84-146 (the restatement's smooth)."""
    keep = A.Keep()
    cls = A.closed_loop_struct(cl, keep)
    wss = A.workspace_struct(ws, keep)
    dw = cl["dw"]
    t = np.ascontiguousarray(t, dtype=np.float64)
    n = t.shape[0]
    arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(n, dw) for a in (pos, vel, ctrl)]
    outs = [np.zeros((n, dw)) for _ in range(3)]
    out3 = np.zeros(3)
    L = lib()
    L.oracle_smooth.argtypes = [C.c_void_p, C.c_void_p, C.c_int] + [C.c_void_p] * 4 + \
        [C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_double, C.c_int] + [C.c_void_p] * 4
    _check(L.oracle_smooth(C.byref(cls), C.byref(wss), n, _p(t), *[_p(a) for a in arrs], plan_mc, alpha, n_mc,
                           C.c_uint64(seed), eps_cc, workers, *[_p(o) for o in outs], _p(out3)))
    return {"traj_pos": outs[0], "traj_vel": outs[1], "traj_ctrl": outs[2], "cost": float(out3[0]),
            "mc": float(out3[1]), "s": float(out3[2])}


def connect(ap, av, bp, bv, tau_max):
    dw = len(ap)
    arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (ap, av, bp, bv)]
    o = np.zeros(3)
    a0, j = np.zeros(dw), np.zeros(dw)
    _check(lib().oracle_connect(dw, *[_p(x) for x in arr], tau_max, _p(o), _p(a0), _p(j)))
    return {"ok": bool(o[0]), "tau": o[1], "cost": o[2], "acc0": a0, "jerk": j}


def steer_cost(ap, av, bp, bv, tau):
    arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (ap, av, bp, bv)]
    return lib().oracle_steer_cost(len(ap), *[_p(x) for x in arr], tau)


def point_free(ws, y):
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    return bool(lib().oracle_point_free(C.byref(s), _p(keep.f64(y))))


def segment_collides(ws, p0, p1):
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    return bool(lib().oracle_segment_collides(C.byref(s), _p(keep.f64(p0)), _p(keep.f64(p1))))


def motion_collides(ws, fp, fv, tp, tv, tau, acc0, jerk, eps_cc):
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    out = C.c_int()
    _check(lib().oracle_motion_collides(C.byref(s), *[_p(keep.f64(x)) for x in (fp, fv, tp, tv)], tau,
                                        _p(keep.f64(acc0)), _p(keep.f64(jerk)), eps_cc, C.byref(out)))
    return bool(out.value)


def local_convex_region(ws, y, ydot, cap=4096):
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    dw = len(y)
    a, b, fb = np.zeros((cap, dw)), np.zeros(cap), np.zeros(cap, dtype=np.uint8)
    n = C.c_int()
    _check(lib().oracle_local_convex_region(C.byref(s), _p(keep.f64(y)), _p(keep.f64(ydot)), cap, _p(a), _p(b),
                                            _p(fb), C.byref(n)))
    k = n.value
    return a[:k], b[:k], fb[:k].astype(bool)


# ------------------------------------------------------------------- graph
class Graph:
    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib().oracle_graph_free(self.h)
            self.h = None

    def export(self) -> dict:
        v = A.GraphViewC()
        lib().oracle_graph_counts(self.h, C.byref(v))
        return A.export_view(v, A.GRAPH_ARRAYS, lib().oracle_graph_export, self.h)


def build_graph(pos, vel, ws, goal, r_n, dt, eps_cc, tau_max, workers=1) -> Graph:
    keep = A.Keep()
    pos = keep.f64(pos)
    vel = keep.f64(vel)
    n, dw = pos.shape
    wss = A.workspace_struct(ws, keep)
    gs = A.goal_struct(goal, keep)
    h = C.c_void_p()
    _check(lib().oracle_build_graph(n, dw, _p(pos), _p(vel), C.byref(wss), C.byref(gs), r_n, dt, eps_cc, tau_max,
                                    workers, C.byref(h)))
    return Graph(h.value)


def graph_from_arrays(g: dict) -> Graph:
    keep = A.Keep()
    v = A.view_from_arrays(A.GraphViewC, g, A.GRAPH_ARRAYS, keep,
                           {k: g[k] for k in ("n_nodes", "dw", "n_edges", "n_waypoints", "n_halfspaces", "n_goal",
                                              "r_n", "dt")})
    h = C.c_void_p()
    _check(lib().oracle_graph_from_view(C.byref(v), C.byref(h)))
    return Graph(h.value)


# ----------------------------------------------------------------- explore
def _params(alpha_min, alpha_max, lam, r_n):
    p = A.ExploreParamsC()
    p.alpha_min, p.alpha_max, p.lambda_, p.r_n = alpha_min, alpha_max, lam, r_n
    return p


def explore(graph: Graph, bank: np.ndarray, alpha_min, alpha_max, lam, r_n, workers=1, masks=True) -> dict:
    bank = np.ascontiguousarray(bank, dtype=np.float64)
    p = _params(alpha_min, alpha_max, lam, r_n)
    h = C.c_void_p()
    _check(lib().oracle_explore(graph.h, bank.shape[1], bank.shape[0] - 1, bank.shape[2], _p(bank), C.byref(p),
                                workers, C.byref(h)))
    try:
        v = A.ExploreViewC()
        lib().oracle_explore_counts(h, C.byref(v))
        out = A.export_view(v, A.EXPLORE_ARRAYS, lib().oracle_explore_export, h,
                            skip=() if masks else ("masks",))
    finally:
        lib().oracle_explore_free(h)
    out["termination"] = A.TERMINATION[out["termination"]]
    return out


def explore_invariants(graph: Graph, bank, alpha_min, alpha_max, lam, r_n):
    bank = np.ascontiguousarray(bank, dtype=np.float64)
    p = _params(alpha_min, alpha_max, lam, r_n)
    counts = np.zeros(4, dtype=np.int64)
    _check(lib().oracle_explore_invariants(graph.h, bank.shape[1], bank.shape[0] - 1, bank.shape[2], _p(bank),
                                           C.byref(p), _p(counts)))
    return dict(zip(["dominance", "double_expansions", "cp", "rounds"], counts.tolist()))


def explore_trace(graph: Graph, bank, alpha_min, alpha_max, lam, r_n) -> list[dict]:
    """The reference RoundHook's view after every round (planner.hpp:245):
    round, expanded ids, arena size, statistics and every node's Pareto set."""
    bank = np.ascontiguousarray(bank, dtype=np.float64)
    p = _params(alpha_min, alpha_max, lam, r_n)
    L = lib()
    L.oracle_explore_trace.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_int64, C.c_void_p]
    n = C.c_int64()
    args = (graph.h, bank.shape[1], bank.shape[0] - 1, bank.shape[2], _p(bank), C.byref(p))
    _check(L.oracle_explore_trace(*args, None, 0, C.byref(n)))
    buf = np.zeros(max(1, n.value), dtype=np.int64)
    _check(L.oracle_explore_trace(*args, _p(buf), n.value, C.byref(n)))
    out, k = [], 0
    while k < n.value:
        rnd, ne = int(buf[k]), int(buf[k + 1])
        k += 2
        exp = buf[k:k + ne].copy()
        k += ne
        n_plans, pp, dcp, rem, dh, nn = (int(x) for x in buf[k:k + 6])
        k += 6
        sizes = buf[k:k + nn]
        k += nn
        tot = int(sizes.sum())
        ids = buf[k:k + tot].copy()
        k += tot
        ptr = np.zeros(nn + 1, dtype=np.int64)
        ptr[1:] = np.cumsum(sizes)
        out.append({"round": rnd, "expanded": exp, "n_plans": n_plans, "partial_plans": pp, "discarded_cp": dcp,
                    "removed_dominated": rem, "discarded_horizon": dh, "pareto_ptr": ptr, "pareto_ids": ids})
    return out


# ---------------------------------------------------------------- pipeline
def scenario_nodes(json_text: str):
    n = C.c_int()
    _check(lib().oracle_scenario_nodes(json_text.encode(), 0, None, None, C.byref(n)))
    m = n.value
    _cl, sc = scenario_models(json_text)
    import json as _json
    dw = len(_json.loads(json_text)["workspace"]["bounds"]["lo"])
    pos, vel = np.zeros((m, dw)), np.zeros((m, dw))
    _check(lib().oracle_scenario_nodes(json_text.encode(), m, _p(pos), _p(vel), C.byref(n)))
    return pos, vel


def run_pump(json_text: str, workers: int = 1, prebuilt: Graph | None = None) -> dict:
    h = C.c_void_p()
    _check(lib().oracle_run_pump(json_text.encode(), workers, prebuilt.h if prebuilt else None, C.byref(h)))
    try:
        s = A.ResultSummaryC()
        lib().oracle_result_summary(h, C.byref(s))
        dw = s.dw
        path = np.zeros(s.path_len, dtype=np.int32)
        pc, pcp = np.zeros(s.n_pareto), np.zeros(s.n_pareto)
        ids, mcs = np.zeros(s.n_mc_evals, dtype=np.int32), np.zeros(s.n_mc_evals)
        n = s.n_traj_points
        tt, tp, tv, tu = np.zeros(n), np.zeros((n, dw)), np.zeros((n, dw)), np.zeros((n, dw))
        lib().oracle_result_arrays(h, *[_p(x) if x.size else None for x in (path, pc, pcp, ids, mcs, tt, tp, tv, tu)])
    finally:
        lib().oracle_result_free(h)
    out = {f: getattr(s, f) for f, _ in s._fields_}
    out.update(path=path, pareto_cost=pc, pareto_cp=pcp, mc_eval_ids=ids, mc_eval_values=mcs, traj_t=tt,
               traj_pos=tp, traj_vel=tv, traj_ctrl=tu)
    out["termination"] = A.TERMINATION[out["termination"]]
    return out


def repeated_rrt(json_text: str, trials: int = 0, alpha: float = -1.0, n_mc: int = 0, workers: int = 1) -> dict:
    """rrt.hpp:50-147 on the scenario (trials / alpha / n_mc <= defaults: the scenario's)."""
    import json as _json

    dw = len(_json.loads(json_text)["workspace"]["bounds"]["lo"])
    L = lib()
    L.oracle_repeated_rrt.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_int, C.c_int] + [C.c_void_p] * 2 + \
        [C.c_int32] + [C.c_void_p] * 5
    out3, out2, n = np.zeros(3), np.zeros(2, dtype=np.int32), C.c_int32()
    _check(L.oracle_repeated_rrt(json_text.encode(), trials, alpha, n_mc, workers, _p(out3), _p(out2), 0, None, None,
                                 None, None, C.byref(n)))
    m = n.value
    t, pos, vel, u = np.zeros(m), np.zeros((m, dw)), np.zeros((m, dw)), np.zeros((m, dw))
    _check(L.oracle_repeated_rrt(json_text.encode(), trials, alpha, n_mc, workers, _p(out3), _p(out2), m, _p(t),
                                 _p(pos), _p(vel), _p(u), C.byref(n)))
    return {"success": bool(out3[0]), "cost": float(out3[1]), "certified_cp": float(out3[2]),
            "trials_reaching_goal": int(out2[0]), "certification_attempts": int(out2[1]),
            "traj_t": t, "traj_pos": pos, "traj_vel": vel, "traj_ctrl": u}
