"""GPU parity of graph build (K_graph), the explore wavefront (K_hsmc +
dominance + frontier compaction) and the full run_pump pipeline against the
CPU oracle, through the C ABI.

Bar: bit-exact edges (cost/tau/coefficients/half-spaces compared by bit
pattern), bit-exact plan arenas (head, parent, cost, cp_hat, t_end, masks),
identical Pareto sets, goal plans, statistics and selected plan; certified CP
and costs bit-identical.
"""
import json
import os

import numpy as np
import pytest

from conftest import scenario_text

pytestmark = pytest.mark.gpu

WORKERS = max(1, min(16, os.cpu_count() or 4))


def ws_of(j):
    w = j["workspace"]
    dw = len(w["bounds"]["lo"])
    obs = w.get("obstacles", [])
    return {"bounds_lo": w["bounds"]["lo"], "bounds_hi": w["bounds"]["hi"],
            "obs_lo": np.array([o["lo"] for o in obs], float).reshape(-1, dw),
            "obs_hi": np.array([o["hi"] for o in obs], float).reshape(-1, dw)}


def goal_of(j):
    return {"lo": j["goal"]["lo"], "hi": j["goal"]["hi"], "max_speed": j["goal"].get("max_speed", 0.0)}


def with_samples(name, samples=None, **kw):
    j = json.loads(scenario_text(name))
    if samples is not None:
        j["samples"] = samples
    j.update(kw)
    return json.dumps(j)


def assert_graph_equal(a, b):
    for k in ("n_nodes", "dw", "n_edges", "n_waypoints", "n_halfspaces", "n_goal"):
        assert a[k] == b[k], k
    for k in ("row_ptr", "edge_to", "edge_nsteps", "edge_wp_off", "wp_hs_off", "hs_fallback", "goal_nodes"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("edge_cost", "edge_tau", "edge_acc0", "edge_jerk", "hs_a", "hs_b"):
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


GRAPH_CASES = [("minimal", None), ("three_obstacle", 300), ("indoor", 400), ("quad3d_three_obstacle", 500),
               ("quad3d_indoor", 600), ("quad3d_forest", 500)]  # forest: 200 boxes (multi-pass regions)


@pytest.mark.parametrize("name,samples", GRAPH_CASES)
def test_build_graph_bit_exact(oracle_lib, gpu_ctx, name, samples):
    from paper_1607_06886_b200 import api

    txt = with_samples(name, samples)
    j = json.loads(txt)
    _, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    og = oracle_lib.build_graph(pos, vel, *args, workers=WORKERS).export()
    gg = api.build_graph(pos, vel, *args, ctx=gpu_ctx).export()
    assert og["n_edges"] > 0
    assert_graph_equal(gg, og)


@pytest.mark.parametrize("n_boxes,samples", [(17, 400), (40, 500), (129, 400), (256, 400), (300, 500), (1000, 400)])
def test_build_graph_many_obstacles(oracle_lib, gpu_ctx, n_boxes, samples):
    """17-256 boxes: grouped region scan (k-d groups of <= 8 boxes); > 256 boxes: the motion cull keeps a
    candidate index list instead of the bitmask and regions take the plain scan."""
    import sys

    from paper_1607_06886_b200 import api

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scenarios"))
    import make_scenarios

    j = make_scenarios.forest(n_boxes=n_boxes)
    j["samples"] = samples
    txt = json.dumps(j)
    _, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    og = oracle_lib.build_graph(pos, vel, *args, workers=WORKERS).export()
    gg = api.build_graph(pos, vel, *args, ctx=gpu_ctx).export()
    assert og["n_edges"] > 0
    assert_graph_equal(gg, og)


@pytest.mark.parametrize("n_boxes,samples", [(40, 600), (300, 500)])
def test_build_graph_2d_many_boxes(oracle_lib, gpu_ctx, n_boxes, samples):
    """2-D worlds above 16 boxes: the spatially ordered region pass and its per-warp distance bounds for dw = 2
    (k_wp_prep / k_regions_once<2, 8> and, above 256 boxes, <2, 128>), small boxes scattered over the 2-D indoor
    world."""
    from paper_1607_06886_b200 import api

    j = json.loads(scenario_text("indoor"))
    rng = np.random.default_rng(7)
    obs = list(j["workspace"]["obstacles"])
    start, glo, ghi = np.array(j["start"]["position"]), np.array(j["goal"]["lo"]), np.array(j["goal"]["hi"])
    while len(obs) < n_boxes:
        c = rng.uniform([0.5, 0.5], [19.5, 11.5])
        e = rng.uniform(0.1, 0.4, size=2)
        lo, hi = c - e / 2, c + e / 2
        if np.all(lo - 0.8 <= start) and np.all(start <= hi + 0.8):
            continue
        if np.all(lo - 0.8 <= ghi) and np.all(glo <= hi + 0.8):
            continue
        obs.append({"lo": [round(float(x), 6) for x in lo], "hi": [round(float(x), 6) for x in hi]})
    j["workspace"]["obstacles"] = obs
    j["samples"] = samples
    txt = json.dumps(j)
    _, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    og = oracle_lib.build_graph(pos, vel, *args, workers=WORKERS).export()
    gg = api.build_graph(pos, vel, *args, ctx=gpu_ctx).export()
    assert og["n_edges"] > 0 and og["n_halfspaces"] > 0
    assert_graph_equal(gg, og)


def test_build_graph_duplicate_boxes(oracle_lib, gpu_ctx):
    """Grouped regions with distance ties: every box listed twice (equal squared distances, the lower
    workspace index must win as in nearest_obstacle_vector's strict first minimum, geom.hpp:128-141) and
    boxes sharing faces."""
    import sys

    from paper_1607_06886_b200 import api

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scenarios"))
    import make_scenarios

    j = make_scenarios.forest(n_boxes=60)
    obs = j["workspace"]["obstacles"]
    # a second copy of each box, interleaved so duplicates land in different k-d groups or the same one
    twins = [dict(o) for o in obs[::-1]]
    faces = [{"lo": [o["hi"][0], o["lo"][1], o["lo"][2]], "hi": [o["hi"][0] + 0.5, o["hi"][1], o["hi"][2]]}
             for o in obs[:20]]
    j["workspace"]["obstacles"] = obs + twins + faces
    j["samples"] = 400
    txt = json.dumps(j)
    _, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    og = oracle_lib.build_graph(pos, vel, *args, workers=WORKERS).export()
    gg = api.build_graph(pos, vel, *args, ctx=gpu_ctx).export()
    assert og["n_edges"] > 0 and og["n_halfspaces"] > 0
    assert_graph_equal(gg, og)


def test_build_graph_degenerate_and_complete(oracle_lib, gpu_ctx):
    """test_plan.cpp:82-101: tiny radius -> no edges; huge radius -> complete."""
    from paper_1607_06886_b200 import api

    ws = {"bounds_lo": [-10.0, -10.0], "bounds_hi": [10.0, 10.0]}
    goal = {"lo": [100.0, 100.0], "hi": [101.0, 101.0], "max_speed": 0.0}
    pos = np.array([[0.0, 0], [5, 0], [9, 0]])
    vel = np.zeros((3, 2))
    assert api.build_graph(pos, vel, ws, goal, 1e-6, 0.1, 0.05, 200.0, ctx=gpu_ctx).edge_count == 0
    g = api.build_graph(pos, vel, ws, goal, 1e6, 0.1, 0.05, 200.0, ctx=gpu_ctx).export()
    assert g["n_edges"] == 6
    assert np.array_equal(np.diff(g["edge_wp_off"]), g["edge_nsteps"])
    with pytest.raises(ValueError):
        api.build_graph(pos, vel, ws, goal, 0.0, 0.1, 0.05, 200.0, ctx=gpu_ctx)


def random_graph_nodes(seed, n, obstacles):
    """test_plan.cpp:58-78 random_zero_noise_graph node generator."""
    import oracle

    pos, vel = [[-8.0, -8.0]], [[0.0, 0.0]]
    ws = {"bounds_lo": [-10.0, -10.0], "bounds_hi": [10.0, 10.0], "obs_lo": [o[0] for o in obstacles],
          "obs_hi": [o[1] for o in obstacles]}
    for i in range(n):
        p = [18 * oracle.uniform(seed, i, 0, 0) - 9, 18 * oracle.uniform(seed, i, 0, 1) - 9]
        v = [2 * oracle.uniform(seed, i, 1, 0) - 1, 2 * oracle.uniform(seed, i, 1, 1) - 1]
        if not oracle.point_free(ws, p):
            continue
        pos.append(p)
        vel.append(v)
    return np.array(pos), np.array(vel), ws


def explore_equal(a, b, masks=True):
    for k in ("n_plans", "n_pareto", "n_goal_plans", "partial_plans", "discarded_cp", "removed_dominated",
              "discarded_horizon", "rounds", "termination"):
        assert a[k] == b[k], (k, a[k], b[k])
    for k in ("head", "parent", "t_end", "pareto_ptr", "pareto_ids", "goal_plans"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("cost", "cp_hat"):
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k
    if masks:
        assert np.array_equal(a["masks"], b["masks"])


@pytest.mark.parametrize("seed", [777, 200, 201])
def test_explore_random_worlds(oracle_lib, gpu_ctx, seed):
    """test_plan.cpp:188-227 setting (noisy bank, alpha band), records equal."""
    from paper_1607_06886_b200 import api

    obstacles = [([-1.0, -4.0], [1.0, 6.0])]
    pos, vel, ws = random_graph_nodes(seed, 80, obstacles)
    goal = {"lo": [5.0, 5.0], "hi": [9.0, 9.0], "max_speed": 0.6}
    scn = {"workspace": {"bounds": {"lo": [-10, -10], "hi": [10, 10]},
                         "obstacles": [{"lo": o[0], "hi": o[1]} for o in obstacles]},
           "start": {"position": [-8, -8]}, "goal": {"lo": [5, 5], "hi": [9, 9], "max_speed": 0.6},
           "noise": {"process": [0, 0, 0.02, 0.02], "measurement": 0.01, "initial": 0.005},
           "dt": 0.25, "samples": 10, "alpha": 0.05}
    cl, _ = oracle_lib.scenario_models(json.dumps(scn))
    og = oracle_lib.build_graph(pos, vel, ws, goal, 9.0, 0.25, 0.05, 200.0, workers=WORKERS)
    gg = api.build_graph(pos, vel, ws, goal, 9.0, 0.25, 0.05, 200.0, ctx=gpu_ctx)
    assert_graph_equal(gg.export(), og.export())
    bank = api.presample_bank(cl, 2048, 64, 9, ctx=gpu_ctx)
    ref = oracle_lib.explore(og, bank, 0.01, 0.2, 0.5, 9.0, workers=WORKERS)
    got = api.explore(gg, 0.01, 0.2, 0.5, 9.0, ctx=gpu_ctx)
    assert ref["n_plans"] > 100
    explore_equal(got, ref)


@pytest.mark.parametrize("name,samples", [("minimal", None), ("three_obstacle", None),
                                          ("quad3d_three_obstacle", 700), ("indoor", 500)])
def test_explore_scenarios(oracle_lib, gpu_ctx, name, samples):
    from paper_1607_06886_b200 import api

    txt = with_samples(name, samples)
    j = json.loads(txt)
    cl, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    og = oracle_lib.build_graph(pos, vel, *args, workers=WORKERS)
    gg = api.build_graph(pos, vel, *args, ctx=gpu_ctx)
    bank = api.presample_bank(cl, j.get("bank_horizon", 2048), j.get("particles", 128), 1, ctx=gpu_ctx)
    eta = sc["eta"]
    amin, amax = sc["alpha"] / eta, min(1.0, eta * sc["alpha"])
    ref = oracle_lib.explore(og, bank, amin, amax, sc["lambda"], sc["r_n"], workers=WORKERS)
    got = api.explore(gg, amin, amax, sc["lambda"], sc["r_n"], ctx=gpu_ctx)
    explore_equal(got, ref)


def test_explore_trivial_and_disconnected(oracle_lib, gpu_ctx):
    """test_plan.cpp:160-186: start inside the goal; unreachable goal."""
    from paper_1607_06886_b200 import api

    zero = {"d": 4, "dw": 2, "F": np.eye(8), "Gv": np.zeros((8, 4)), "Gw": np.zeros((8, 2)), "Sv": np.zeros((4, 4)),
            "Sw": np.zeros((2, 2)), "S0": np.zeros((4, 4)), "C": np.hstack([np.eye(2), np.zeros((2, 2))])}
    api.presample_bank(zero, 64, 8, 1, ctx=gpu_ctx)
    ws = {"bounds_lo": [-10.0, -10.0], "bounds_hi": [10.0, 10.0]}
    pos = np.array([[0.0, 0.0], [5.0, 5.0]])
    vel = np.zeros((2, 2))
    g = api.build_graph(pos, vel, ws, {"lo": [-1, -1], "hi": [1, 1], "max_speed": 0.1}, 1e6, 0.25, 0.05, 200.0,
                        ctx=gpu_ctx)
    r = api.explore(g, 0.5, 1.0, 0.5, 1e6, ctx=gpu_ctx)
    assert r["termination"] == "goal_below_alpha_min"
    assert r["cost"][r["goal_plans"][0]] == 0.0
    g2 = api.build_graph(pos, vel, ws, {"lo": [100, 100], "hi": [101, 101], "max_speed": 0.0}, 1e6, 0.25, 0.05,
                         200.0, ctx=gpu_ctx)
    r2 = api.explore(g2, 0.5, 1.0, 0.5, 1e6, ctx=gpu_ctx)
    assert len(r2["goal_plans"]) == 0
    assert r2["termination"] == "frontier_exhausted"


def assert_run_equal(got, ref):
    for k in ("success", "termination", "partial_plans", "path_len", "n_pareto", "n_mc_evals", "n_traj_points"):
        assert got[k] == ref[k], (k, got[k], ref[k])
    for k in ("cost", "certified_cp", "cp_hat", "pre_smoothing_cost", "smoothing_s"):
        assert got[k] == ref[k], (k, got[k], ref[k])
    assert np.array_equal(got["path"], ref["path"])
    assert np.array_equal(got["mc_eval_ids"], ref["mc_eval_ids"])
    assert np.array_equal(got["mc_eval_values"], ref["mc_eval_values"])
    assert np.array_equal(got["pareto_cost"].view(np.uint64), ref["pareto_cost"].view(np.uint64))
    assert np.array_equal(got["pareto_cp"], ref["pareto_cp"])
    for k in ("traj_t", "traj_pos", "traj_vel", "traj_ctrl"):
        assert np.array_equal(got[k].view(np.uint64), ref[k].view(np.uint64)), k


@pytest.mark.parametrize("name,samples,mc", [("minimal", None, 4000), ("three_obstacle", None, 4000),
                                             ("quad3d_three_obstacle", 800, 4000), ("quad3d_forest", 700, 3000)])
def test_run_pump_matches_oracle(oracle_lib, gpu_ctx, name, samples, mc):
    from paper_1607_06886_b200 import api

    txt = with_samples(name, samples, mc_samples=mc)
    got = api.run_pump(api.parse_scenario(txt), ctx=gpu_ctx)
    ref = oracle_lib.run_pump(txt, workers=WORKERS)
    assert_run_equal(got, ref)


def test_run_pump_many_boxes(oracle_lib, gpu_ctx):
    """More than 256 boxes: the list-mode motion cull in collide, the region scan above 256 boxes, and the
    smoothing probes' nominal check with the list-mode warp cull (k_smooth_probe<DW, kCullList>)."""
    import sys

    from paper_1607_06886_b200 import api

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scenarios"))
    import make_scenarios

    j = make_scenarios.forest(n_boxes=300)
    j.update({"samples": 5000, "mc_samples": 3000})  # (reaches the goal and smooths: s = 0.072)
    txt = json.dumps(j)
    got = api.run_pump(api.parse_scenario(txt), ctx=gpu_ctx)
    ref = oracle_lib.run_pump(txt, workers=WORKERS)
    assert_run_equal(got, ref)


def test_run_pump_goal_fallback_sample(oracle_lib, gpu_ctx):
    """sample_free's goal fallback (sample.hpp:63-88): no Halton sample lands in the goal and its centre is blocked
    (the 10-box forest), so the first free goal Halton state is appended; searched on the device."""
    import sys

    from paper_1607_06886_b200 import api

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scenarios"))
    import make_scenarios

    j = make_scenarios.forest(n_boxes=10)
    j.update({"samples": 1500, "mc_samples": 3000})
    j["goal"]["lo"] = [20.0, 20.0, 3.5]  # a 0.3 m goal box is missed by 1500 Halton samples: its free centre is
    j["goal"]["hi"] = [20.3, 20.3, 3.8]  # appended
    txt = json.dumps(j)
    got = api.run_pump(api.parse_scenario(txt), ctx=gpu_ctx)
    ref = oracle_lib.run_pump(txt, workers=WORKERS)
    assert_run_equal(got, ref)
    box = {"lo": [20.1, 20.1, 3.6], "hi": [20.2, 20.2, 3.7]}  # and with the goal centre inside an obstacle
    j["workspace"]["obstacles"] = j["workspace"]["obstacles"] + [box]
    txt = json.dumps(j)
    got = api.run_pump(api.parse_scenario(txt), ctx=gpu_ctx)
    ref = oracle_lib.run_pump(txt, workers=WORKERS)
    assert_run_equal(got, ref)


@pytest.mark.parametrize("name,samples", [("three_obstacle", None), ("quad3d_three_obstacle", 600)])
def test_run_pump_prebuilt_graph(oracle_lib, gpu_ctx, name, samples):
    """run_pump(s, workers, prebuilt) (pump.hpp:170-171): a graph built from
    the scenario's own node set gives the solve without prebuilt, bit for bit."""
    from paper_1607_06886_b200 import api

    txt = with_samples(name, samples, mc_samples=3000)
    sc = api.parse_scenario(txt)
    pos, vel = sc.nodes()
    p = sc.params()
    g = api.build_graph(pos, vel, sc.workspace(), sc.goal(), p["r_n"], p["dt"], p["eps_cc"], p["tau_max"],
                        ctx=gpu_ctx)
    a = api.run_pump(sc, prebuilt=g, ctx=gpu_ctx)
    b = api.run_pump(sc, ctx=gpu_ctx)
    assert a["path"].tolist() == b["path"].tolist()
    assert a["cost"] == b["cost"] and a["certified_cp"] == b["certified_cp"]
    assert a["partial_plans"] == b["partial_plans"] and a["n_edges"] == b["n_edges"]
    ref = oracle_lib.run_pump(txt, workers=WORKERS)
    assert_run_equal(a, ref)


@pytest.mark.parametrize("world", [2, 3])
def test_graph_row_slices_concatenate(oracle_lib, gpu_ctx, world):
    """SURVEY §8e, graph sharded by source row: the per-rank slices
    (pump_build_graph_rows, what each rank builds before the NCCL gather)
    concatenate to the full graph bit for bit, and row_ptr is their sum."""
    from paper_1607_06886_b200 import api

    txt = with_samples("quad3d_indoor", 500)
    j = json.loads(txt)
    _, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    full = api.build_graph(pos, vel, *args, ctx=gpu_ctx).export()
    n = pos.shape[0]
    parts = []
    for r in range(world):
        lo, hi = api.shard_range(n, r, world)
        parts.append(api.build_graph_rows(pos, vel, *args, lo, hi, ctx=gpu_ctx).export())
    row_ptr = sum(p["row_ptr"].astype(np.int64) for p in parts)
    assert np.array_equal(row_ptr, full["row_ptr"])
    for k in ("edge_to", "edge_nsteps", "hs_fallback"):
        assert np.array_equal(np.concatenate([p[k] for p in parts]), full[k]), k
    for k in ("edge_cost", "edge_tau", "edge_acc0", "edge_jerk", "hs_a", "hs_b"):
        assert np.array_equal(np.concatenate([p[k] for p in parts]).view(np.uint64), full[k].view(np.uint64)), k
    # CSR offsets: each slice starts at 0
    wp, hs, wbase, hbase = [np.zeros(1, np.int64)], [np.zeros(1, np.int64)], 0, 0
    for p in parts:
        wp.append(p["edge_wp_off"][1:] + wbase)
        hs.append(p["wp_hs_off"][1:] + hbase)
        wbase += int(p["edge_wp_off"][-1])
        hbase += int(p["wp_hs_off"][-1])
    assert np.array_equal(np.concatenate(wp), full["edge_wp_off"])
    assert np.array_equal(np.concatenate(hs), full["wp_hs_off"])


def rrt_kat_text(obstacles=()):
    """test_plan.cpp:279-306 setting: empty 2-D world, zero noise."""
    return json.dumps({"name": "rrt_kat", "workspace": {"bounds": {"lo": [-10, -10], "hi": [10, 10]},
                                                        "obstacles": [{"lo": o[0], "hi": o[1]} for o in obstacles]},
                       "start": {"position": [-5, 0], "velocity": [0, 0]},
                       "goal": {"lo": [4, -1], "hi": [6, 1], "max_speed": 0.5},
                       "noise": {"process": [0, 0, 0, 0], "measurement": 0, "initial": 0},
                       "dt": 0.25, "alpha": 0.05, "max_speed": 1.0, "connection_radius": 6.0, "mc_samples": 200,
                       "rrt": {"max_iterations": 80}, "samples": 10})


@pytest.mark.parametrize("case", ["kat", "sealed", "minimal", "three_obstacle", "quad3d_three_obstacle"])
def test_repeated_rrt_matches_oracle(oracle_lib, gpu_ctx, case):
    """rrt.hpp:50-147 (the Table 1 baseline) on the GPU: trials reaching the
    goal, certification attempts, cost, certified CP and trajectory bits."""
    from paper_1607_06886_b200 import api

    if case == "kat":
        txt, trials, n_mc = rrt_kat_text(), 40, 200
    elif case == "sealed":
        txt, trials, n_mc = rrt_kat_text([([3, -3], [7, 3])]), 20, 200
    else:
        txt, trials, n_mc = with_samples(case, None, mc_samples=2000), 64, 2000
    alpha = json.loads(txt).get("alpha", 0.05)
    got = api.repeated_rrt(api.parse_scenario(txt), trials, alpha, n_mc, ctx=gpu_ctx)
    ref = oracle_lib.repeated_rrt(txt, trials, alpha, n_mc, workers=WORKERS)
    for k in ("success", "trials_reaching_goal", "certification_attempts"):
        assert got[k] == ref[k], (k, got[k], ref[k])
    assert got["cost"] == ref["cost"] and got["certified_cp"] == ref["certified_cp"]
    assert np.array_equal(got["traj_t"], ref["traj_t"])
    for k in ("traj_pos", "traj_vel", "traj_ctrl"):
        assert np.array_equal(got[k].view(np.uint64), ref[k].view(np.uint64)), k
    if case == "kat":
        assert got["success"]
    if case == "sealed":
        assert not got["success"]
