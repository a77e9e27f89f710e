"""Oracle vs the literal reference code (CPU).

oracle/_ref/libpumpref.so is the reference's own headers
(/root/reference/proj/include, compiled in place by oracle/ref/Makefile)
over the Eigen-subset shim (include/compat).  With glibc normals on both
sides, the oracle restatement must reproduce the reference's bank bits, and
every output of run_pump, bit for bit.  This pins the restatement's control
flow (sampling, graph, explore, dominance, termination, bisection,
smoothing) against the reference source.  Model-synthesis arithmetic comes
from the same linalg routines on both sides; Eigen's own rounding stays
unpinned.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import ROOT, scenario_text

REF = os.path.join(ROOT, "oracle", "_ref", "libpumpref.so")
pytestmark = pytest.mark.skipif(not os.path.exists(REF), reason="reference not built (needs /root/reference)")


def ref():
    L = C.CDLL(REF)
    L.ref_last_error.restype = C.c_char_p
    L.ref_presample_bank.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_ulonglong, C.c_int, C.c_void_p]
    L.ref_closed_loop_F.argtypes = [C.c_char_p, C.c_void_p]
    L.ref_run_pump.argtypes = [C.c_char_p, C.c_int] + [C.c_void_p] * 11
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def variant(name, **kw):
    j = json.loads(scenario_text(name))
    j.update(kw)
    return json.dumps(j)


def ref_run(L, text, workers):
    sc = np.zeros(8)
    path = np.zeros(4096, dtype=np.int32)
    ids, vals = np.zeros(4096, dtype=np.int32), np.zeros(4096)
    ne, npar, nt = C.c_int(), C.c_int(), C.c_int()
    pc, pp = np.zeros(4096), np.zeros(4096)
    tt, tp = np.zeros(100000), np.zeros(300000)
    rc = L.ref_run_pump(text.encode(), workers, _p(sc), _p(path), _p(ids), _p(vals), C.byref(ne), _p(pc), _p(pp),
                        C.byref(npar), _p(tt), _p(tp), C.byref(nt))
    assert rc == 0, L.ref_last_error()
    dw = len(json.loads(text)["workspace"]["bounds"]["lo"])
    return {"success": int(sc[0]), "cost": sc[1], "certified_cp": sc[2], "cp_hat": sc[3],
            "partial_plans": int(sc[4]), "smoothing_s": sc[5], "pre_smoothing_cost": sc[6],
            "path": path[:int(sc[7])].tolist(), "mc_eval_ids": ids[:ne.value].tolist(),
            "mc_eval_values": vals[:ne.value].tolist(), "pareto_cost": pc[:npar.value],
            "pareto_cp": pp[:npar.value], "traj_t": tt[:nt.value], "traj_pos": tp[:nt.value * dw].reshape(-1, dw)}


@pytest.mark.parametrize("name", ["minimal", "quad3d_indoor"])
def test_closed_loop_matches_reference(oracle_lib, name):
    L = ref()
    txt = scenario_text(name)
    cl, _ = oracle_lib.scenario_models(txt)
    F = np.zeros_like(cl["F"])
    assert L.ref_closed_loop_F(txt.encode(), _p(F)) == 0
    assert np.array_equal(F.view(np.uint64), cl["F"].view(np.uint64))


@pytest.mark.parametrize("name,T,n", [("minimal", 40, 512), ("quad3d_three_obstacle", 80, 32)])
def test_bank_bits_match_reference_glibc(oracle_lib, name, T, n):
    L = ref()
    txt = scenario_text(name)
    cl, _ = oracle_lib.scenario_models(txt)
    dw = cl["dw"]
    out = np.zeros((T + 1, n, dw))
    assert L.ref_presample_bank(txt.encode(), T, n, 7, 4, _p(out)) == 0
    oracle_lib.set_normal_mode(oracle_lib.GLIBC)
    try:
        ob = oracle_lib.presample_bank(cl, T, n, 7, workers=4)
    finally:
        oracle_lib.set_normal_mode(oracle_lib.PORTABLE)
    assert np.array_equal(out.view(np.uint64), ob.view(np.uint64))


@pytest.mark.parametrize("name,kw", [("minimal", {"mc_samples": 2000}),
                                     ("three_obstacle", {"mc_samples": 2000}),
                                     ("quad3d_three_obstacle", {"samples": 500, "mc_samples": 2000})])
def test_run_pump_matches_reference(oracle_lib, name, kw):
    L = ref()
    txt = variant(name, **kw)
    workers = min(8, os.cpu_count() or 2)
    r = ref_run(L, txt, workers)
    for mode in (oracle_lib.GLIBC, oracle_lib.PORTABLE):
        oracle_lib.set_normal_mode(mode)
        try:
            o = oracle_lib.run_pump(txt, workers=workers)
        finally:
            oracle_lib.set_normal_mode(oracle_lib.PORTABLE)
        # decisions (node path, front, probes) agree in both normal modes
        assert o["path"].tolist() == r["path"], mode
        assert o["partial_plans"] == r["partial_plans"]
        assert o["mc_eval_ids"].tolist() == r["mc_eval_ids"]
        assert np.array_equal(o["pareto_cost"], r["pareto_cost"])
        assert np.array_equal(o["pareto_cp"], r["pareto_cp"])
        if mode == oracle_lib.GLIBC:  # the literal reference: every bit
            assert o["cost"] == r["cost"] and o["certified_cp"] == r["certified_cp"]
            assert o["mc_eval_values"].tolist() == r["mc_eval_values"]
            assert o["smoothing_s"] == r["smoothing_s"]
            assert np.array_equal(o["traj_t"], r["traj_t"])
            assert np.array_equal(o["traj_pos"].view(np.uint64), r["traj_pos"].view(np.uint64))


def rrt_kat_text(obstacles=()):
    """test_plan.cpp:279-306 setting: empty 2-D world, zero noise."""
    return json.dumps({"name": "rrt_kat", "workspace": {"bounds": {"lo": [-10, -10], "hi": [10, 10]},
                                                        "obstacles": [{"lo": o[0], "hi": o[1]} for o in obstacles]},
                       "start": {"position": [-5, 0], "velocity": [0, 0]},
                       "goal": {"lo": [4, -1], "hi": [6, 1], "max_speed": 0.5},
                       "noise": {"process": [0, 0, 0, 0], "measurement": 0, "initial": 0},
                       "dt": 0.25, "alpha": 0.05, "max_speed": 1.0, "connection_radius": 6.0, "mc_samples": 200,
                       "rrt": {"max_iterations": 80}, "samples": 10})


@pytest.mark.parametrize("case", ["kat", "minimal", "three_obstacle"])
def test_repeated_rrt_matches_reference(oracle_lib, case):
    """rrt.hpp:50-147: the oracle's repeated_rrt reproduces the literal
    reference (glibc normals for the MC certification) bit for bit."""
    L = ref()
    L.ref_repeated_rrt.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_int, C.c_int] + [C.c_void_p] * 2 + \
        [C.c_int] + [C.c_void_p] * 2
    if case == "kat":
        txt, trials, n_mc = rrt_kat_text(), 40, 200
    else:
        txt, trials, n_mc = variant(case, mc_samples=2000), 60, 2000
    alpha = json.loads(txt).get("alpha", 0.05)
    workers = min(8, os.cpu_count() or 2)
    o4, o2 = np.zeros(4), np.zeros(2, dtype=np.int32)
    tt, tp = np.zeros(100000), np.zeros(300000)
    rc = L.ref_repeated_rrt(txt.encode(), trials, alpha, n_mc, workers, _p(o4), _p(o2), 100000, _p(tt), _p(tp))
    assert rc == 0, L.ref_last_error()
    oracle_lib.set_normal_mode(oracle_lib.GLIBC)
    try:
        o = oracle_lib.repeated_rrt(txt, trials, alpha, n_mc, workers=workers)
    finally:
        oracle_lib.set_normal_mode(oracle_lib.PORTABLE)
    assert o["success"] == bool(o4[0])
    assert o["trials_reaching_goal"] == o2[0] and o["certification_attempts"] == o2[1]
    assert o["cost"] == o4[1] and o["certified_cp"] == o4[2]
    n = int(o4[3])
    dw = len(json.loads(txt)["workspace"]["bounds"]["lo"])
    assert np.array_equal(o["traj_t"], tt[:n])
    assert np.array_equal(o["traj_pos"].view(np.uint64), tp[:n * dw].reshape(-1, dw).view(np.uint64))
    if case == "kat":
        assert o["success"] and o["trials_reaching_goal"] > 0
