"""Python mirror of the reference ``pump`` API over ``libpump_gpu.so``.

Names and argument meanings follow the reference headers
(/root/reference/proj/include/pump/*.hpp): ``presample_bank`` (lti.hpp:257),
``hsmc_extend`` (cp.hpp:180), ``mc_certify`` (cp.hpp:214), ``build_graph``
(graph.hpp:50), ``explore`` (planner.hpp:74), ``run_pump`` (pump.hpp:170),
``load_scenario`` / ``parse_scenario`` (scenario.hpp:144-269).  Errors map to
the reference's exception types: ``ValueError`` <- std::invalid_argument,
``IndexError`` <- std::out_of_range, ``ScenarioError`` <- pump::ScenarioError,
``RuntimeError`` <- std::runtime_error.

Every call runs on the GPU through the C ABI; there is no CPU fallback: if
the library or a B200 is missing, calls raise ``PumpCudaError``.
"""
from __future__ import annotations

import ctypes as C
import json as _json
import os

import numpy as np

from . import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpump_gpu.so")

_lib = None


class PumpError(RuntimeError):
    pass


class ScenarioError(PumpError):
    pass


class PumpCudaError(PumpError):
    pass


class CapacityError(PumpError):
    pass


class LibraryMissing(ImportError):
    pass


_EXC = {A.PUMP_E_INVALID_ARGUMENT: ValueError, A.PUMP_E_OUT_OF_RANGE: IndexError,
        A.PUMP_E_RUNTIME: RuntimeError, A.PUMP_E_SCENARIO: ScenarioError, A.PUMP_E_CUDA: PumpCudaError,
        A.PUMP_E_CAPACITY: CapacityError, A.PUMP_E_LOGIC: RuntimeError,
        A.PUMP_E_HOOK: RuntimeError}

# every symbol include/pump_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "pump_last_error", "pump_abi_version", "pump_ctx_create", "pump_ctx_destroy", "pump_ctx_last_kernel_ms",
    "pump_ctx_launch_count", "pump_scenario_parse", "pump_scenario_load", "pump_scenario_free",
    "pump_scenario_closed_loop", "pump_scenario_params", "pump_presample_bank", "pump_bank_upload",
    "pump_hsmc_extend_batch", "pump_explore_run_hooked", "pump_smooth", "pump_mc_certify_batch", "pump_mc_certify", "pump_build_graph", "pump_graph_upload",
    "pump_graph_counts", "pump_graph_export", "pump_graph_free", "pump_explore_run", "pump_explore_counts",
    "pump_explore_export", "pump_explore_free", "pump_run", "pump_result_summary_get", "pump_result_arrays",
    "pump_result_free", "pump_nccl_unique_id", "pump_ctx_set_comm", "pump_ctx_set_collectives", "pump_shard_range", "pump_ctx_profile",
    "pump_ctx_profile_read", "pump_ctx_io_bytes", "pump_ctx_flush_l2", "pump_peak_fp64", "pump_ctx_stream",
    "pump_scenario_nodes", "pump_build_graph_rows", "pump_rrt_run", "pump_probe_round_latency",
]


def lib():
    """Load libpump_gpu.so (raises LibraryMissing loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                                 "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.pump_last_error.restype = C.c_char_p
        L.pump_ctx_last_kernel_ms.restype = C.c_double
        L.pump_ctx_last_kernel_ms.argtypes = [vp]
        L.pump_ctx_launch_count.restype = C.c_int64
        L.pump_ctx_launch_count.argtypes = [vp]
        L.pump_ctx_create.argtypes = [C.c_int, vp]
        L.pump_ctx_destroy.argtypes = [vp]
        L.pump_scenario_parse.argtypes = [C.c_char_p, vp]
        L.pump_scenario_load.argtypes = [C.c_char_p, vp]
        L.pump_scenario_free.argtypes = [vp]
        L.pump_scenario_closed_loop.argtypes = [vp] * 10
        L.pump_scenario_params.argtypes = [vp, vp, vp]
        L.pump_presample_bank.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_uint64, vp]
        L.pump_bank_upload.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp]
        L.pump_hsmc_extend_batch.argtypes = [vp, C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pump_mc_certify_batch.argtypes = [vp, vp, vp, C.c_int32, vp, vp, C.c_int64, C.c_int64, C.c_uint64,
                                            C.c_double, vp]
        L.pump_mc_certify.argtypes = [vp, vp, vp, C.c_int32, vp, C.c_int32, C.c_uint64, C.c_double, vp]
        if hasattr(L, "pump_build_graph"):
            L.pump_build_graph.argtypes = [vp, C.c_int32, C.c_int32, vp, vp, vp, vp, C.c_double, C.c_double,
                                           C.c_double, C.c_double, vp]
            L.pump_graph_upload.argtypes = [vp, vp, vp]
            L.pump_graph_counts.argtypes = [vp, vp]
            L.pump_graph_export.argtypes = [vp, vp]
            L.pump_graph_free.argtypes = [vp]
            L.pump_explore_run.argtypes = [vp, vp, vp, vp]
            L.pump_explore_counts.argtypes = [vp, vp]
            L.pump_explore_export.argtypes = [vp, vp]
            L.pump_explore_free.argtypes = [vp]
            L.pump_run.argtypes = [vp, vp, vp, vp]
            L.pump_result_summary_get.argtypes = [vp, vp]
            L.pump_result_arrays.argtypes = [vp] * 10
            L.pump_result_free.argtypes = [vp]
        L.pump_nccl_unique_id.argtypes = [vp]
        L.pump_ctx_set_comm.argtypes = [vp, C.c_int, C.c_int, vp]
        L.pump_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, vp, vp]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().pump_last_error().decode()
        exc = _EXC.get(rc, PumpError)
        e = exc(msg)
        e.code = rc
        raise e


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream + resident bank (``pump_ctx``)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().pump_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().pump_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def last_kernel_ms(self) -> float:
        return lib().pump_ctx_last_kernel_ms(self.h)

    def io_counters(self) -> dict:
        """pump_ctx_io_bytes: H2D / D2H bytes, MC rollout-steps, device
        allocations, collectives issued."""
        b = np.zeros(5, dtype=np.int64)
        lib().pump_ctx_io_bytes(self.h, _p(b))
        return dict(zip(("h2d_bytes", "d2h_bytes", "mc_rollout_steps", "device_allocs", "collectives"),
                        b.tolist()))

    @property
    def launches(self) -> int:
        return lib().pump_ctx_launch_count(self.h)


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_ctx


# ----------------------------------------------------------------- scenario
class Scenario:
    """Parsed scenario (scenario.hpp:34-77) held by the library."""

    def __init__(self, handle, text: str | None):
        self.h = handle
        self.text = text

    @staticmethod
    def parse(text: str) -> "Scenario":
        h = C.c_void_p()
        _check(lib().pump_scenario_parse(text.encode(), C.byref(h)))
        return Scenario(h, text)

    @staticmethod
    def load(path: str) -> "Scenario":
        h = C.c_void_p()
        _check(lib().pump_scenario_load(path.encode(), C.byref(h)))
        with open(path) as f:
            text = f.read()
        return Scenario(h, text)

    def __del__(self):
        if getattr(self, "h", None):
            lib().pump_scenario_free(self.h)
            self.h = None

    def closed_loop(self) -> dict:
        d, dw = C.c_int32(), C.c_int32()
        _check(lib().pump_scenario_closed_loop(self.h, C.byref(d), C.byref(dw), *([None] * 7)))
        d, dw = d.value, dw.value
        m = {"F": np.zeros((2 * d, 2 * d)), "Gv": np.zeros((2 * d, d)), "Gw": np.zeros((2 * d, dw)),
             "Sv": np.zeros((d, d)), "Sw": np.zeros((dw, dw)), "S0": np.zeros((d, d)), "C": np.zeros((dw, d))}
        _check(lib().pump_scenario_closed_loop(self.h, C.byref(C.c_int32()), C.byref(C.c_int32()),
                                               *[_p(m[k]) for k in ("F", "Gv", "Gw", "Sv", "Sw", "S0", "C")]))
        m["d"], m["dw"] = d, dw
        return m

    def params(self) -> dict:
        f = np.zeros(8)
        i = np.zeros(8, dtype=np.int64)
        _check(lib().pump_scenario_params(self.h, _p(f), _p(i)))
        keys_f = ["eps_cc", "r_n", "tau_max", "alpha", "eta", "lambda", "dt", "max_speed"]
        keys_i = ["samples", "particles", "mc_samples", "bank_horizon", "seed_bank", "seed_mc", "seed_rrt", "dw"]
        out = dict(zip(keys_f, f.tolist()))
        out.update(dict(zip(keys_i, [int(x) for x in i])))
        return out

    def nodes(self):
        """(pos, vel), n x dw each: the node set run_pump plans over."""
        L = lib()
        L.pump_scenario_nodes.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        n = C.c_int32()
        _check(L.pump_scenario_nodes(self.h, 0, None, None, C.byref(n)))
        dw = self.params()["dw"]
        pos, vel = np.zeros((n.value, dw)), np.zeros((n.value, dw))
        _check(L.pump_scenario_nodes(self.h, n.value, _p(pos), _p(vel), C.byref(n)))
        return pos, vel

    def goal(self) -> dict:
        j = _json.loads(self.text)
        g = j["goal"]
        return {"lo": np.array(g["lo"], float), "hi": np.array(g["hi"], float),
                "max_speed": float(g.get("max_speed", 0.0))}  # scenario.hpp default

    def workspace(self) -> dict:
        j = _json.loads(self.text)
        ws = j["workspace"]
        obs = ws.get("obstacles", [])
        dw = len(ws["bounds"]["lo"])
        return {"bounds_lo": np.array(ws["bounds"]["lo"], float), "bounds_hi": np.array(ws["bounds"]["hi"], float),
                "obs_lo": np.array([o["lo"] for o in obs], float).reshape(-1, dw),
                "obs_hi": np.array([o["hi"] for o in obs], float).reshape(-1, dw)}


def parse_scenario(text: str) -> Scenario:
    return Scenario.parse(text)


def load_scenario(path: str) -> Scenario:
    return Scenario.load(path)


# --------------------------------------------------------------------- bank
def presample_bank(cl: dict, t_max: int, n: int, seed: int, ctx: Context | None = None,
                   copy_out: bool = True):
    """presample_bank (lti.hpp:257-292) on the GPU; returns dy[(t_max+1), n, dw]
    (the bank also stays resident in ``ctx`` for hsmc_extend / explore)."""
    ctx = ctx or default_context()
    keep = A.Keep()
    s = A.closed_loop_struct(cl, keep)
    out = np.zeros((t_max + 1, n, cl["dw"])) if copy_out else None
    _check(lib().pump_presample_bank(ctx.h, C.byref(s), t_max, n, C.c_uint64(seed), _p(out)))
    return out


def bank_upload(dy: np.ndarray, ctx: Context | None = None):
    ctx = ctx or default_context()
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    _check(lib().pump_bank_upload(ctx.h, dy.shape[1], dy.shape[0] - 1, dy.shape[2], _p(dy)))


# --------------------------------------------------------------------- hsmc
def hsmc_extend_batch(masks_in, step_off, step_t, step_hs_off, hs_a, hs_b, ctx: Context | None = None):
    """Batched hsmc_extend (cp.hpp:180-208) against the context's bank."""
    ctx = ctx or default_context()
    masks_in = np.ascontiguousarray(masks_in, dtype=np.uint64)
    n_tasks, n_words = masks_in.shape
    arrs = [np.ascontiguousarray(step_off, dtype=np.int64), np.ascontiguousarray(step_t, dtype=np.int32),
            np.ascontiguousarray(step_hs_off, dtype=np.int64),
            np.ascontiguousarray(hs_a, dtype=np.float64).reshape(-1), np.ascontiguousarray(hs_b, dtype=np.float64)]
    arrs = [a if a.size else np.zeros(1, a.dtype) for a in arrs]
    out = np.zeros_like(masks_in)
    pop = np.zeros(n_tasks, dtype=np.int32)
    _check(lib().pump_hsmc_extend_batch(ctx.h, n_tasks, n_words, _p(masks_in), *[_p(a) for a in arrs], _p(out),
                                        _p(pop)))
    return out, pop


def full_mask(n: int) -> np.ndarray:
    """ParticleMask::full (cp.hpp:24-31)."""
    w = np.full((n + 63) // 64, np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    if n % 64:
        w[-1] = np.uint64((1 << (n % 64)) - 1)
    return w


def hsmc_extend(mask: np.ndarray, steps, n_particles: int, ctx: Context | None = None):
    """Single hsmc_extend with the reference's signature semantics.  steps is a
    list of (t, region) with region a list of (a, b) half-spaces or None.
    Returns (mask', cp)."""
    step_t, hs_off, a_rows, b_rows = [], [0], [], []
    for t, region in steps:
        step_t.append(t)
        for a, b in (region or []):
            a_rows.append(np.asarray(a, float))
            b_rows.append(float(b))
        hs_off.append(len(b_rows))
    dw = a_rows[0].size if a_rows else 1
    out, pop = hsmc_extend_batch(np.asarray(mask, np.uint64)[None, :], [0, len(steps)], step_t, hs_off,
                                 np.array(a_rows).reshape(-1, dw) if a_rows else np.zeros((0, dw)),
                                 np.array(b_rows), ctx)
    return out[0], 1.0 - float(pop[0]) / n_particles


# ----------------------------------------------------------------------- mc
def mc_certify_batch(cl: dict, ws: dict, trajectories, rollout_lo: int, rollout_hi: int, seed: int,
                     eps_cc: float, ctx: Context | None = None) -> np.ndarray:
    """Colliding-rollout counts of rollouts [lo, hi) for every trajectory."""
    ctx = ctx or default_context()
    keep = A.Keep()
    cls = A.closed_loop_struct(cl, keep)
    wss = A.workspace_struct(ws, keep)
    dw = cl["dw"]
    ys = [np.asarray(t, float).reshape(-1, dw) for t in trajectories]
    off = np.zeros(len(ys) + 1, dtype=np.int64)
    off[1:] = np.cumsum([y.shape[0] for y in ys])
    y = np.ascontiguousarray(np.concatenate(ys, axis=0) if ys else np.zeros((1, dw)))
    hits = np.zeros(len(ys), dtype=np.int64)
    _check(lib().pump_mc_certify_batch(ctx.h, C.byref(cls), C.byref(wss), len(ys), _p(off), _p(y), rollout_lo,
                                       rollout_hi, C.c_uint64(seed), eps_cc, _p(hits)))
    return hits


def smooth(t, pos, vel, ctrl, plan_mc: float, alpha: float, cl: dict, ws: dict, n_mc: int, seed: int,
           eps_cc: float, ctx: Context | None = None) -> dict:
    """smooth (pump.hpp:84-146) of a plan trajectory on the device (the
    speculative bisection chain run_pump uses): {traj_pos, traj_vel,
    traj_ctrl, cost, mc, s}; times are the plan's."""
    ctx = ctx or default_context()
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
    L.pump_smooth.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32] + [C.c_void_p] * 4 + \
        [C.c_double, C.c_double, C.c_int32, C.c_uint64, C.c_double] + [C.c_void_p] * 4
    _check(L.pump_smooth(ctx.h, C.byref(cls), C.byref(wss), n, _p(t), *[_p(a) for a in arrs], plan_mc, alpha, n_mc,
                         C.c_uint64(seed), eps_cc, *[_p(o) for o in outs], _p(out3)))
    return {"traj_pos": outs[0], "traj_vel": outs[1], "traj_ctrl": outs[2], "cost": float(out3[0]),
            "mc": float(out3[1]), "s": float(out3[2])}


def mc_certify(y_nom, cl: dict, ws: dict, n_mc: int, seed: int, eps_cc: float, ctx: Context | None = None) -> float:
    """mc_certify (cp.hpp:214-268): fraction of colliding rollouts."""
    if n_mc < 1:
        raise ValueError("mc_certify: need at least one rollout")
    if len(y_nom) == 0:
        raise ValueError("mc_certify: empty trajectory")
    return float(mc_certify_batch(cl, ws, [y_nom], 0, n_mc, seed, eps_cc, ctx)[0]) / n_mc


# -------------------------------------------------------------------- graph
class Graph:
    """Device-resident SampleGraph (graph.hpp:25-37)."""

    def __init__(self, handle, ctx):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            lib().pump_graph_free(self.h)
            self.h = None

    def counts(self) -> dict:
        v = A.GraphViewC()
        _check(lib().pump_graph_counts(self.h, C.byref(v)))
        return {f: getattr(v, f) for f, _ in v._fields_ if f not in A.GRAPH_ARRAYS}

    def export(self) -> dict:
        v = A.GraphViewC()
        _check(lib().pump_graph_counts(self.h, C.byref(v)))
        return A.export_view(v, A.GRAPH_ARRAYS, lambda h, pv: lib().pump_graph_export(h, pv), self.h)

    @property
    def edge_count(self) -> int:
        return int(self.counts()["n_edges"])


def build_graph(pos, vel, ws: dict, goal: dict, r_n: float, dt: float, eps_cc: float, tau_max: float,
                ctx: Context | None = None) -> Graph:
    """build_graph (graph.hpp:50-95) on the GPU for nodes (pos, vel: n x dw)."""
    ctx = ctx or default_context()
    keep = A.Keep()
    pos = keep.f64(pos)
    vel = keep.f64(vel)
    n, dw = pos.shape
    wss = A.workspace_struct(ws, keep)
    gs = A.goal_struct(goal, keep)
    h = C.c_void_p()
    _check(lib().pump_build_graph(ctx.h, n, dw, _p(pos), _p(vel), C.byref(wss), C.byref(gs), r_n, dt, eps_cc,
                                  tau_max, C.byref(h)))
    return Graph(h, ctx)


def build_graph_rows(pos, vel, ws: dict, goal: dict, r_n: float, dt: float, eps_cc: float, tau_max: float,
                     row_lo: int, row_hi: int, ctx: Context | None = None) -> Graph:
    """The edges of source rows [row_lo, row_hi) only: one rank's slice of the
    multi-GPU graph build (pump_build_graph_rows)."""
    ctx = ctx or default_context()
    keep = A.Keep()
    pos = keep.f64(pos)
    vel = keep.f64(vel)
    n, dw = pos.shape
    wss = A.workspace_struct(ws, keep)
    gs = A.goal_struct(goal, keep)
    h = C.c_void_p()
    L = lib()
    L.pump_build_graph_rows.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32,
                                        C.c_int32, C.c_void_p]
    _check(L.pump_build_graph_rows(ctx.h, n, dw, _p(pos), _p(vel), C.byref(wss), C.byref(gs), r_n, dt, eps_cc,
                                   tau_max, row_lo, row_hi, C.byref(h)))
    return Graph(h, ctx)


def graph_upload(g: dict, ctx: Context | None = None) -> Graph:
    """Upload a prebuilt graph (flat arrays as returned by Graph.export)."""
    ctx = ctx or default_context()
    keep = A.Keep()
    v = A.view_from_arrays(A.GraphViewC, g, A.GRAPH_ARRAYS, keep,
                           {k: g[k] for k in ("n_nodes", "dw", "n_edges", "n_waypoints", "n_halfspaces", "n_goal",
                                              "r_n", "dt")})
    h = C.c_void_p()
    _check(lib().pump_graph_upload(ctx.h, C.byref(v), C.byref(h)))
    return Graph(h, ctx)


# ------------------------------------------------------------------ explore
ROUND_HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_int32), C.c_int64)


def _explore_state(h, masks: bool) -> dict:
    v = A.ExploreViewC()
    _check(lib().pump_explore_counts(h, C.byref(v)))
    out = A.export_view(v, A.EXPLORE_ARRAYS, lambda hh, pv: lib().pump_explore_export(hh, pv), h,
                        skip=() if masks else ("masks",))
    out["termination"] = A.TERMINATION[out["termination"]]
    return out


def explore(graph: Graph, alpha_min: float, alpha_max: float, lam: float, r_n: float,
            ctx: Context | None = None, masks: bool = True, hook=None) -> dict:
    """explore (planner.hpp:74-267) on the context's resident bank.

    hook(round, state, expanded) is the reference's RoundHook
    (planner.hpp:51-52, 245): called after every round with the exploration
    state so far (the same dict this function returns, goal_plans empty) and
    the ids the round expanded; rounds then run one at a time.  An exception
    raised by the hook stops the run and is re-raised here."""
    ctx = ctx or graph.ctx
    p = A.ExploreParamsC()
    p.alpha_min, p.alpha_max, p.lambda_, p.r_n = alpha_min, alpha_max, lam, r_n
    h = C.c_void_p()
    if hook is None:
        _check(lib().pump_explore_run(ctx.h, graph.h, C.byref(p), C.byref(h)))
    else:
        err = []

        def tramp(_user, rnd, state, expanded, n_exp):
            try:
                st = _explore_state(state, masks)
                st["termination"] = ""
                hook(int(rnd), st, np.ctypeslib.as_array(expanded, (int(n_exp),)).copy() if n_exp else
                     np.zeros(0, np.int32))
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised after the run stops
                err.append(e)
                return 1

        cb = ROUND_HOOK(tramp)
        L = lib()
        L.pump_explore_run_hooked.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, ROUND_HOOK, C.c_void_p,
                                              C.c_void_p]
        rc = L.pump_explore_run_hooked(ctx.h, graph.h, C.byref(p), cb, None, C.byref(h))
        if err:
            raise err[0]
        _check(rc)
    try:
        out = _explore_state(h, masks)
    finally:
        lib().pump_explore_free(h)
    return out


# ----------------------------------------------------------------- pipeline
def run_pump(scenario: Scenario, prebuilt: Graph | None = None, ctx: Context | None = None) -> dict:
    """run_pump (pump.hpp:170-263): graph build, bank + explore, bisection
    selection with MC certification, smoothing — all hot loops on the GPU."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().pump_run(ctx.h, scenario.h, prebuilt.h if prebuilt else None, C.byref(h)))
    try:
        s = A.ResultSummaryC()
        _check(lib().pump_result_summary_get(h, C.byref(s)))
        dw = s.dw
        path = np.zeros(s.path_len, dtype=np.int32)
        pc, pcp = np.zeros(s.n_pareto), np.zeros(s.n_pareto)
        ids, mcs = np.zeros(s.n_mc_evals, dtype=np.int32), np.zeros(s.n_mc_evals)
        n = s.n_traj_points
        tt, tp, tv, tu = np.zeros(n), np.zeros((n, dw)), np.zeros((n, dw)), np.zeros((n, dw))
        _check(lib().pump_result_arrays(h, *[_p(x) if x.size else None
                                             for x in (path, pc, pcp, ids, mcs, tt, tp, tv, tu)]))
    finally:
        lib().pump_result_free(h)
    out = {f: getattr(s, f) for f, _ in s._fields_}
    out.update(path=path, pareto_cost=pc, pareto_cp=pcp, mc_eval_ids=ids, mc_eval_values=mcs, traj_t=tt,
               traj_pos=tp, traj_vel=tv, traj_ctrl=tu)
    out["termination"] = A.TERMINATION[out["termination"]]
    return out


def repeated_rrt(scenario: Scenario, trials: int = 0, alpha: float = -1.0, n_mc: int = 0,
                 ctx: Context | None = None) -> dict:
    """repeated_rrt (rrt.hpp:50-147) on the GPU: success, cost, certified_cp,
    trials_reaching_goal, certification_attempts and the trajectory.  Zero /
    negative arguments take the scenario's rrt.trials / alpha / mc_samples."""
    ctx = ctx or default_context()
    L = lib()
    L.pump_rrt_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_int32, C.c_void_p]
    h = C.c_void_p()
    _check(L.pump_rrt_run(ctx.h, scenario.h, trials, alpha, n_mc, C.byref(h)))
    try:
        s = A.ResultSummaryC()
        _check(L.pump_result_summary_get(h, C.byref(s)))
        dw, n = s.dw, s.n_traj_points
        tt, tp, tv, tu = np.zeros(n), np.zeros((n, dw)), np.zeros((n, dw)), np.zeros((n, dw))
        _check(L.pump_result_arrays(h, None, None, None, None, None, *[_p(x) if x.size else None
                                                                       for x in (tt, tp, tv, tu)]))
    finally:
        L.pump_result_free(h)
    return {"success": bool(s.success), "cost": s.cost, "certified_cp": s.certified_cp,
            "trials_reaching_goal": s.rrt_trials_reaching_goal,
            "certification_attempts": s.rrt_certification_attempts,
            "traj_t": tt, "traj_pos": tp, "traj_vel": tv, "traj_ctrl": tu}


# ---------------------------------------------------------------- multi-GPU
def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rollouts [lo, hi) owned by `rank` of `world` (the library's partition)."""
    return n * rank // world, n * (rank + 1) // world


def set_comm(ctx: Context, rank: int, world: int, group=None):
    """Shard the MC certification of pump_run across `world` ranks (one GPU
    each): rank 0 creates the NCCL id, torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist

    buf = np.zeros(128, dtype=np.uint8)
    if rank == 0:
        _check(lib().pump_nccl_unique_id(_p(buf)))
    t = torch.from_numpy(buf.astype(np.int64)).cuda() if dist.get_backend(group) == "nccl" else \
        torch.from_numpy(buf.astype(np.int64))
    dist.broadcast(t, src=0, group=group)
    buf = t.cpu().numpy().astype(np.uint8)
    _check(lib().pump_ctx_set_comm(ctx.h, rank, world, _p(buf)))


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.c_int64)
GATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                        C.c_int32)


def set_collectives(ctx: Context, rank: int, world: int, group=None):
    """The same sharding as set_comm over the torch.distributed process
    group's own collectives (any backend, e.g. gloo) instead of NCCL: the
    library stages the int64 hit counts / graph row slices through host
    memory and calls back into dist.all_reduce / dist.all_gather.  Several
    ranks may share one GPU this way (nothing on the device waits for another
    rank); used by the multi-rank tests on a single B200."""
    import torch
    import torch.distributed as dist

    def allreduce(_user, values, count):
        try:
            a = np.ctypeslib.as_array(values, (int(count),))
            t = torch.from_numpy(a.copy())
            dist.all_reduce(t, group=group)
            a[:] = t.numpy()
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed collective
            return 1

    def gather(_user, send, recv, off, length, n_ranks):
        try:
            offs = np.ctypeslib.as_array(off, (int(n_ranks),)).copy()
            lens = np.ctypeslib.as_array(length, (int(n_ranks),)).copy()
            m = int(lens.max()) if n_ranks else 0
            mine = np.zeros(max(m, 1), np.uint8)
            if lens[rank]:
                mine[:lens[rank]] = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), (int(lens[rank]),))
            parts = [torch.zeros(max(m, 1), dtype=torch.uint8) for _ in range(int(n_ranks))]
            dist.all_gather(parts, torch.from_numpy(mine), group=group)
            total = int((offs + lens).max())
            out = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), (max(total, 1),))
            for r in range(int(n_ranks)):
                out[offs[r]:offs[r] + lens[r]] = parts[r].numpy()[:lens[r]]
            return 0
        except Exception:  # noqa: BLE001
            return 1

    ctx._coll = (ALLREDUCE_FN(allreduce), GATHER_FN(gather))  # keep the callbacks alive with the context
    L = lib()
    L.pump_ctx_set_collectives.argtypes = [C.c_void_p, C.c_int, C.c_int, ALLREDUCE_FN, GATHER_FN, C.c_void_p]
    _check(L.pump_ctx_set_collectives(ctx.h, rank, world, ctx._coll[0], ctx._coll[1], None))


# ------------------------------------------------------- host-side helpers
# The reference's scalar geometry / steering functions, evaluated on the host
# by the same __host__ __device__ code the kernels run (pump_gpu.h "host
# helpers"); no GPU needed.
def _host_lib():
    L = lib()
    if not getattr(L, "_host_typed", False):
        vp, d, i32 = C.c_void_p, C.c_double, C.c_int32
        L.pump_connect.argtypes = [i32, vp, vp, vp, vp, d, vp, vp, vp]
        L.pump_steer_cost.argtypes = [i32, vp, vp, vp, vp, d]
        L.pump_steer_cost.restype = d
        L.pump_point_free.argtypes = [vp, vp]
        L.pump_motion_collides.argtypes = [vp, vp, vp, vp, vp, d, vp, vp, d, vp]
        L.pump_local_convex_region.argtypes = [vp, vp, vp, i32, vp, vp, vp, vp]
        L._host_typed = True
    return L


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def connect(ap, av, bp, bv, tau_max):
    """steer.hpp:111-182 (connect): {'ok', 'tau', 'cost', 'acc0', 'jerk'}."""
    arr = [_f64(x) for x in (ap, av, bp, bv)]
    dw = arr[0].size
    o, a0, j = np.zeros(3), np.zeros(dw), np.zeros(dw)
    _check(_host_lib().pump_connect(dw, *[_p(x) for x in arr], tau_max, _p(o), _p(a0), _p(j)))
    return {"ok": bool(o[0]), "tau": o[1], "cost": o[2], "acc0": a0, "jerk": j}


def steer_cost(ap, av, bp, bv, tau):
    """steer.hpp:84-94."""
    arr = [_f64(x) for x in (ap, av, bp, bv)]
    return _host_lib().pump_steer_cost(arr[0].size, *[_p(x) for x in arr], tau)


def point_free(ws: dict, y) -> bool:
    """geom.hpp:56-61."""
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    return bool(_host_lib().pump_point_free(C.byref(s), _p(keep.f64(y))))


def motion_collides(ws: dict, fp, fv, tp, tv, tau, acc0, jerk, eps_cc) -> bool:
    """geom.hpp:96-123."""
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    out = C.c_int32()
    _check(_host_lib().pump_motion_collides(C.byref(s), *[_p(keep.f64(x)) for x in (fp, fv, tp, tv)], tau,
                                            _p(keep.f64(acc0)), _p(keep.f64(jerk)), eps_cc, C.byref(out)))
    return bool(out.value)


def local_convex_region(ws: dict, y, ydot, cap: int = 4096):
    """geom.hpp:189-225: (a [n, dw], b [n], fallback [n])."""
    keep = A.Keep()
    s = A.workspace_struct(ws, keep)
    yy = keep.f64(y)
    dw = yy.size
    a, b, fb = np.zeros((cap, dw)), np.zeros(cap), np.zeros(cap, dtype=np.uint8)
    n = C.c_int32()
    _check(_host_lib().pump_local_convex_region(C.byref(s), _p(yy), _p(keep.f64(ydot)), cap, _p(a), _p(b), _p(fb),
                                                C.byref(n)))
    k = n.value
    return a[:k], b[:k], fb[:k].astype(bool)
