"""ctypes mirror of the POD structs in include/pump_gpu.h.

Only layouts and small numpy helpers live here; the product entry points are
bound in ``paper_1607_06886_b200.api`` and the test-only oracle in
``oracle``.  Keeping the layouts in one place guarantees both sides exchange
byte-identical inputs.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

PUMP_OK = 0
PUMP_E_INVALID_ARGUMENT = 1
PUMP_E_OUT_OF_RANGE = 2
PUMP_E_RUNTIME = 3
PUMP_E_SCENARIO = 4
PUMP_E_CUDA = 5
PUMP_E_CAPACITY = 6
PUMP_E_LOGIC = 7
PUMP_E_HOOK = 8

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


class ClosedLoopC(C.Structure):
    _fields_ = [("d", C.c_int32), ("dw", C.c_int32), ("F", _dp), ("Gv", _dp), ("Gw", _dp),
                ("Sv", _dp), ("Sw", _dp), ("S0", _dp), ("C", _dp)]


class WorkspaceC(C.Structure):
    _fields_ = [("dw", C.c_int32), ("n_obs", C.c_int32), ("bounds_lo", _dp), ("bounds_hi", _dp),
                ("obs_lo", _dp), ("obs_hi", _dp)]


class GoalC(C.Structure):
    _fields_ = [("lo", _dp), ("hi", _dp), ("max_speed", C.c_double)]


class GraphViewC(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("dw", C.c_int32),
                ("n_edges", C.c_int64), ("n_waypoints", C.c_int64), ("n_halfspaces", C.c_int64),
                ("n_goal", C.c_int32), ("r_n", C.c_double), ("dt", C.c_double),
                ("node_pos", _dp), ("node_vel", _dp), ("row_ptr", _i64p), ("edge_to", _i32p),
                ("edge_cost", _dp), ("edge_tau", _dp), ("edge_acc0", _dp), ("edge_jerk", _dp),
                ("edge_nsteps", _i32p), ("edge_wp_off", _i64p), ("wp_hs_off", _i64p),
                ("hs_a", _dp), ("hs_b", _dp), ("hs_fallback", _u8p), ("goal_nodes", _i32p)]


class ExploreParamsC(C.Structure):
    _fields_ = [("alpha_min", C.c_double), ("alpha_max", C.c_double), ("lambda_", C.c_double),
                ("r_n", C.c_double)]


class ExploreViewC(C.Structure):
    _fields_ = [("n_plans", C.c_int64), ("n_words", C.c_int32), ("n_nodes", C.c_int32),
                ("n_pareto", C.c_int64), ("n_goal_plans", C.c_int64),
                ("partial_plans", C.c_int64), ("discarded_cp", C.c_int64),
                ("removed_dominated", C.c_int64), ("discarded_horizon", C.c_int64),
                ("rounds", C.c_int32), ("termination", C.c_int32),
                ("head", _i32p), ("parent", _i32p), ("cost", _dp), ("cp_hat", _dp), ("t_end", _i32p),
                ("masks", _u64p), ("pareto_ptr", _i64p), ("pareto_ids", _i32p), ("goal_plans", _i32p)]


class ResultSummaryC(C.Structure):
    _fields_ = [("success", C.c_int32), ("termination", C.c_int32),
                ("path_len", C.c_int32), ("n_pareto", C.c_int32), ("n_mc_evals", C.c_int32),
                ("n_traj_points", C.c_int32), ("dw", C.c_int32),
                ("partial_plans", C.c_int64),
                ("cost", C.c_double), ("certified_cp", C.c_double), ("cp_hat", C.c_double),
                ("pre_smoothing_cost", C.c_double), ("smoothing_s", C.c_double),
                ("build_graph_seconds", C.c_double), ("explore_seconds", C.c_double),
                ("selection_seconds", C.c_double),
                ("bank_ms", C.c_double), ("explore_kernel_ms", C.c_double), ("mc_ms", C.c_double),
                ("n_edges", C.c_int64), ("n_plans", C.c_int64), ("mc_rollouts", C.c_int64),
                ("rrt_trials_reaching_goal", C.c_int32), ("rrt_certification_attempts", C.c_int32),
                ("explore_hs_read", C.c_int64)]


TERMINATION = {0: "goal_below_alpha_min", 1: "frontier_exhausted"}


def ptr(a: np.ndarray | None, ctype=C.c_double):
    """Pointer to a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


class Keep:
    """Holds numpy buffers alive while a ctypes struct points into them."""

    def __init__(self):
        self.refs = []

    def f64(self, x):
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        self.refs.append(a)
        return a


def closed_loop_struct(cl: dict, keep: Keep) -> ClosedLoopC:
    s = ClosedLoopC()
    s.d, s.dw = int(cl["d"]), int(cl["dw"])
    for k in ("F", "Gv", "Gw", "Sv", "Sw", "S0", "C"):
        setattr(s, k, ptr(keep.f64(cl[k])))
    return s


def workspace_struct(ws: dict, keep: Keep) -> WorkspaceC:
    s = WorkspaceC()
    lo = keep.f64(ws["bounds_lo"])
    s.dw = lo.size
    s.bounds_lo = ptr(lo)
    s.bounds_hi = ptr(keep.f64(ws["bounds_hi"]))
    olo = keep.f64(np.asarray(ws.get("obs_lo", []), dtype=np.float64).reshape(-1, lo.size))
    ohi = keep.f64(np.asarray(ws.get("obs_hi", []), dtype=np.float64).reshape(-1, lo.size))
    s.n_obs = olo.shape[0]
    s.obs_lo = ptr(olo) if olo.size else None
    s.obs_hi = ptr(ohi) if ohi.size else None
    return s


def goal_struct(goal: dict, keep: Keep) -> GoalC:
    s = GoalC()
    s.lo = ptr(keep.f64(goal["lo"]))
    s.hi = ptr(keep.f64(goal["hi"]))
    s.max_speed = float(goal["max_speed"])
    return s


GRAPH_ARRAYS = {
    # name: (dtype, ctype, size-fn(view))
    "node_pos": (np.float64, C.c_double, lambda v: v.n_nodes * v.dw),
    "node_vel": (np.float64, C.c_double, lambda v: v.n_nodes * v.dw),
    "row_ptr": (np.int64, C.c_int64, lambda v: v.n_nodes + 1),
    "edge_to": (np.int32, C.c_int32, lambda v: v.n_edges),
    "edge_cost": (np.float64, C.c_double, lambda v: v.n_edges),
    "edge_tau": (np.float64, C.c_double, lambda v: v.n_edges),
    "edge_acc0": (np.float64, C.c_double, lambda v: v.n_edges * v.dw),
    "edge_jerk": (np.float64, C.c_double, lambda v: v.n_edges * v.dw),
    "edge_nsteps": (np.int32, C.c_int32, lambda v: v.n_edges),
    "edge_wp_off": (np.int64, C.c_int64, lambda v: v.n_edges + 1),
    "wp_hs_off": (np.int64, C.c_int64, lambda v: v.n_waypoints + 1),
    "hs_a": (np.float64, C.c_double, lambda v: v.n_halfspaces * v.dw),
    "hs_b": (np.float64, C.c_double, lambda v: v.n_halfspaces),
    "hs_fallback": (np.uint8, C.c_uint8, lambda v: v.n_halfspaces),
    "goal_nodes": (np.int32, C.c_int32, lambda v: v.n_goal),
}

EXPLORE_ARRAYS = {
    "head": (np.int32, C.c_int32, lambda v: v.n_plans),
    "parent": (np.int32, C.c_int32, lambda v: v.n_plans),
    "cost": (np.float64, C.c_double, lambda v: v.n_plans),
    "cp_hat": (np.float64, C.c_double, lambda v: v.n_plans),
    "t_end": (np.int32, C.c_int32, lambda v: v.n_plans),
    "masks": (np.uint64, C.c_uint64, lambda v: v.n_plans * v.n_words),
    "pareto_ptr": (np.int64, C.c_int64, lambda v: v.n_nodes + 1),
    "pareto_ids": (np.int32, C.c_int32, lambda v: v.n_pareto),
    "goal_plans": (np.int32, C.c_int32, lambda v: v.n_goal_plans),
}


def export_view(view, table, exporter, handle, skip=()):
    """Allocate numpy buffers per ``table`` sized from ``view``'s counts, point
    the view at them, call ``exporter(handle, byref(view))`` and return a dict
    of arrays plus the scalar counts."""
    out = {}
    for name, (dt, ct, size) in table.items():
        if name in skip:
            setattr(view, name, None)
            continue
        a = np.zeros(int(size(view)), dtype=dt)
        out[name] = a
        setattr(view, name, ptr(a, ct) if a.size else C.cast(C.c_void_p(0), C.POINTER(ct)))
        if a.size == 0:
            # keep a valid non-null pointer for empty arrays
            b = np.zeros(1, dtype=dt)
            out["_empty_" + name] = b
            setattr(view, name, ptr(b, ct))
    rc = exporter(handle, C.byref(view))
    if rc != 0:
        raise RuntimeError(f"export failed rc={rc}")
    for f, _ in view._fields_:
        if f not in table:
            out[f] = getattr(view, f)
    for k in [k for k in out if k.startswith("_empty_")]:
        del out[k]
    return out


def view_from_arrays(cls, arrays: dict, table, keep: Keep, scalars: dict):
    """Build a view struct pointing at numpy arrays (for uploads)."""
    v = cls()
    for k, val in scalars.items():
        setattr(v, k, val)
    for name, (dt, ct, _size) in table.items():
        if name not in arrays or arrays[name] is None:
            setattr(v, name, None)
            continue
        a = np.ascontiguousarray(np.asarray(arrays[name], dtype=dt))
        if a.size == 0:
            a = np.zeros(1, dtype=dt)
        keep.refs.append(a)
        setattr(v, name, ptr(a, ct))
    return v
