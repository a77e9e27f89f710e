"""Pin the CPU oracle against the reference's own tests (CPU only).

Each test ports a known-answer / property test of /root/reference/proj/tests
(file:line in the docstring) to the oracle restatement, so the oracle the GPU
is compared with is itself checked against the reference's expectations.
"""
import heapq
import json
import math
import os

import numpy as np
import pytest

import oracle
from conftest import scenario_text

W = max(1, min(8, os.cpu_count() or 2))


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()
    oracle.set_normal_mode(oracle.PORTABLE)
    yield
    oracle.set_normal_mode(oracle.PORTABLE)


# ------------------------------------------------------------------- rng
def test_counter_hash_matches_python_restatement():
    """rng.hpp:8-34 restated in pure Python (arbitrary precision + mask)."""
    M = (1 << 64) - 1

    def mix(x):
        x ^= x >> 30
        x = (x * 0xbf58476d1ce4e5b9) & M
        x ^= x >> 27
        x = (x * 0x94d049bb133111eb) & M
        return x ^ (x >> 31)

    for seed, a, b, c in [(1, 0, 0, 0), (2, 5, 7, 9), (2 ** 63 + 5, 123456, 2 ** 40, 2 << 20)]:
        h = mix((seed + 0x9e3779b97f4a7c15) & M)
        for x in (a, b, c):
            h = mix((h + x) & M)
        assert oracle.counter_hash(seed, a, b, c) == h
        assert oracle.uniform(seed, a, b, c) == ((h >> 11) + 1.0) * 2.0 ** -53


def test_portable_normal_close_to_glibc():
    """The portable normal (pmath.h) differs from glibc's by <= a few ulp;
    agreement rate is reported, not assumed."""
    a = np.arange(20000, dtype=np.uint64)
    oracle.set_normal_mode(oracle.GLIBC)
    g = oracle.normals(1, a, 0, 0)
    oracle.set_normal_mode(oracle.PORTABLE)
    p = oracle.normals(1, a, 0, 0)
    diff_ulp = np.abs(g.view(np.int64) - p.view(np.int64))
    assert diff_ulp.max() <= 4
    assert np.mean(diff_ulp == 0) > 0.7
    assert abs(np.mean(p)) < 0.03 and abs(np.std(p) - 1) < 0.03


# ------------------------------------------------------------ model/bank
def scalar_loop(a, v, s0, w=1.0):
    return {"d": 1, "dw": 1, "F": np.array([[a, 0.0], [0.0, a]]), "Gv": np.array([[1.0], [0.0]]),
            "Gw": np.array([[0.0], [0.0]]), "Sv": np.array([[math.sqrt(v)]]), "Sw": np.array([[math.sqrt(w)]]),
            "S0": np.array([[math.sqrt(s0)]]), "C": np.array([[1.0]])}


def di1d_scenario(process_v, meas_w, s0):
    """A 1-D double-integrator scenario (test_lti.cpp double_integrator_1d)."""
    return json.dumps({"workspace": {"bounds": {"lo": [-100], "hi": [100]}}, "start": {"position": [0]},
                       "goal": {"lo": [50], "hi": [60]}, "dt": 0.1, "samples": 5, "alpha": 0.05,
                       "noise": {"process": [0, process_v], "measurement": meas_w, "initial": s0}})


def test_bank_zero_noise_is_zero():
    """test_lti.cpp:185-195."""
    cl, _ = oracle.scenario_models(di1d_scenario(0.0, 1.0, 0.0))
    cl["Sw"] = np.zeros_like(cl["Sw"])  # no measurement noise in the rollouts either
    assert np.all(oracle.presample_bank(cl, 10, 16, 7) == 0.0)


def test_bank_deterministic_across_workers_and_seeds():
    """test_lti.cpp:197-210."""
    cl, _ = oracle.scenario_models(di1d_scenario(0.05, 0.02, 0.01))
    a = oracle.presample_bank(cl, 12, 37, 42, workers=1)
    b = oracle.presample_bank(cl, 12, 37, 42, workers=3)
    c = oracle.presample_bank(cl, 12, 37, 43, workers=1)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert not np.array_equal(a, c)


def test_bank_covariance_matches_propagation():
    """test_lti.cpp:212-234: empirical variance within 3 sigma of the
    closed-loop covariance recursion (lti.hpp:221-240), N = 1e5."""
    cl, _ = oracle.scenario_models(di1d_scenario(0.02, 0.01, 0.01))
    n, T = 100000, 10
    bank = oracle.presample_bank(cl, T, n, 5, workers=W)
    d = cl["d"]
    sz = np.zeros((2 * d, 2 * d))
    sz[:d, :d] = cl["S0"] @ cl["S0"].T
    vq, wq = cl["Sv"] @ cl["Sv"].T, cl["Sw"] @ cl["Sw"].T
    for t in range(T + 1):
        truth = (cl["C"] @ sz[:d, :d] @ cl["C"].T)[0, 0]
        emp = np.mean(bank[t, :, 0] ** 2)
        assert abs(emp - truth) < 3 * truth * math.sqrt(2.0 / n) + 1e-12
        sz = cl["F"] @ sz @ cl["F"].T + cl["Gv"] @ vq @ cl["Gv"].T + cl["Gw"] @ wq @ cl["Gw"].T


# ----------------------------------------------------------------- steer
def test_connect_rest_to_rest():
    """test_steer.cpp:8-28: tau* = 36^(1/4), cost 3.2660."""
    m = oracle.connect([0.0], [0.0], [1.0], [0.0], 10.0)
    assert m["ok"]
    assert abs(m["tau"] - 36 ** 0.25) < 1e-6
    assert abs(m["cost"] - 3.2660) < 1e-4
    taus = np.arange(1, 1000001) * 1e-5
    best = min(oracle.steer_cost([0.0], [0.0], [1.0], [0.0], t) for t in taus[::50])
    assert m["cost"] <= best + 1e-9


def test_connect_identity_translation_and_reversal():
    """test_steer.cpp:30-47, 72-83."""
    a, av = [1.0, 2.0], [0.3, -0.1]
    i = oracle.connect(a, av, a, av, 10.0)
    assert i["ok"] and i["tau"] == 0.0 and i["cost"] == 0.0
    b, bv = [3.0, -1.0], [-0.2, 0.4]
    m1 = oracle.connect(a, av, b, bv, 50.0)
    m2 = oracle.connect([x + 7.5 for x in a], av, [x + 7.5 for x in b], bv, 50.0)
    assert abs(m1["cost"] - m2["cost"]) < 1e-9 * m1["cost"]
    assert abs(m1["tau"] - m2["tau"]) < 1e-7 * m1["tau"]
    f = oracle.connect([0.0, 1.0], [0.5, -0.3], [2.0, -1.0], [0.1, 0.8], 100.0)
    r = oracle.connect([2.0, -1.0], [-0.1, -0.8], [0.0, 1.0], [-0.5, 0.3], 100.0)
    assert abs(f["cost"] - r["cost"]) < 1e-8 * f["cost"]


def test_connect_random_probes_never_beat_optimum():
    """test_steer.cpp:49-70."""
    for trial in range(30):
        ap = [10 * oracle.uniform(11, trial, 0, k) - 5 for k in range(2)]
        av = [2 * oracle.uniform(11, trial, 1, k) - 1 for k in range(2)]
        bp = [10 * oracle.uniform(11, trial, 2, k) - 5 for k in range(2)]
        bv = [2 * oracle.uniform(11, trial, 3, k) - 1 for k in range(2)]
        m = oracle.connect(ap, av, bp, bv, 100.0)
        assert m["ok"]
        for p in range(40):
            tau = 100.0 * oracle.uniform(11, trial, 4, p)
            assert m["cost"] <= oracle.steer_cost(ap, av, bp, bv, tau) + 1e-9


def test_waypoint_remainder_rule():
    """test_steer.cpp:85-105."""
    a, av, b, bv = [0.0, 0.0], [0.2, 0.0], [1.0, 0.5], [0.0, -0.1]
    f1 = oracle.fixed_time_connect(a, av, b, bv, 1.0)
    t, p, _, _ = oracle.waypoints(a, av, b, bv, f1, 0.25)
    assert len(t) == 5 and t[-1] == 1.0
    assert np.max(np.abs(p[-1] - b)) < 1e-9
    f2 = oracle.fixed_time_connect(a, av, b, bv, 1.1)
    t, p, _, _ = oracle.waypoints(a, av, b, bv, f2, 0.25)
    assert len(t) == 6 and abs(t[4] - 1.0) < 1e-12 and abs(t[5] - 1.1) < 1e-12


# ------------------------------------------------------------------ geom
def box_world(obs):
    return {"bounds_lo": [-10.0, -10.0], "bounds_hi": [10.0, 10.0], "obs_lo": [o[0] for o in obs],
            "obs_hi": [o[1] for o in obs]}


def test_point_free_boundary_rules():
    """test_geom.cpp:25-33."""
    w = box_world([([0, 0], [1, 1])])
    assert oracle.point_free(w, [-5, -5])
    assert not oracle.point_free(w, [0.5, 0.5])
    assert not oracle.point_free(w, [0, 0])
    assert not oracle.point_free(w, [11, 0])
    assert oracle.point_free(box_world([]), [3, 3])


def test_motion_collides_cases_and_resolution():
    """test_geom.cpp:35-85."""
    w = box_world([([-1, -1], [1, 1])])
    m = oracle.connect([-5.0, 0.0], [0.0, 0.0], [5.0, 0.0], [0.0, 0.0], 100.0)
    args = ([-5.0, 0.0], [0.0, 0.0], [5.0, 0.0], [0.0, 0.0], m["tau"], m["acc0"], m["jerk"])
    assert oracle.motion_collides(w, *args, 0.05)
    assert not oracle.motion_collides(box_world([]), *args, 0.05)
    w3 = box_world([([-2, -2], [-0.5, 2]), ([1, -1], [3, 0.5]), ([-4, 4], [4, 6])])
    checked = 0
    for trial in range(100):
        ap = [16 * oracle.uniform(21, trial, 0, k) - 8 for k in range(2)]
        av = [2 * oracle.uniform(21, trial, 1, k) - 1 for k in range(2)]
        bp = [16 * oracle.uniform(21, trial, 2, k) - 8 for k in range(2)]
        bv = [2 * oracle.uniform(21, trial, 3, k) - 1 for k in range(2)]
        m = oracle.connect(ap, av, bp, bv, 200.0)
        if not m["ok"]:
            continue
        checked += 1
        args = (ap, av, bp, bv, m["tau"], m["acc0"], m["jerk"])
        assert oracle.motion_collides(w3, *args, 0.05) == oracle.motion_collides(w3, *args, 0.005)
    assert checked >= 90


def test_local_convex_region_cases_and_pruning():
    """test_geom.cpp:158-213."""
    one = box_world([([2, -1], [3, 1])])
    a, b, fb = oracle.local_convex_region(one, [0.0, 0.0], [0.0, 0.0])
    assert len(b) == 1 and fb.all()
    two = box_world([([2, -1], [3, 1]), ([-4, -1], [-3, 1])])
    a, b, _ = oracle.local_convex_region(two, [0.0, 0.0], [0.0, 0.0])
    assert len(b) == 2 and np.linalg.norm(a[0]) <= np.linalg.norm(a[1])
    with pytest.raises(ValueError):
        oracle.local_convex_region(one, [2.5, 0.0], [0.0, 0.0])
    for trial in range(40):
        obs = []
        for i in range(10):
            cx, cy = 16 * oracle.uniform(25, trial, i, 0) - 8, 16 * oracle.uniform(25, trial, i, 1) - 8
            wx, wy = 0.5 + 2 * oracle.uniform(25, trial, i, 2), 0.5 + 2 * oracle.uniform(25, trial, i, 3)
            obs.append(([cx - wx, cy - wy], [cx + wx, cy + wy]))
        w = box_world(obs)
        y = np.array([16 * oracle.uniform(25, trial, 100, 0) - 8, 16 * oracle.uniform(25, trial, 100, 1) - 8])
        if not oracle.point_free(w, y):
            continue
        a, b, _ = oracle.local_convex_region(w, y, [0.0, 0.0])
        assert len(b) <= 10
        for lo, hi in obs:
            for s in range(50):
                p = np.array([lo[0] + oracle.uniform(26, trial, s, 0) * (hi[0] - lo[0]),
                              lo[1] + oracle.uniform(26, trial, s, 1) * (hi[1] - lo[1])])
                assert any(a[h] @ (p - y) >= b[h] - 1e-9 * (1 + b[h]) for h in range(len(b)))


# ---------------------------------------------------------------- HSMC/MC
def test_hsmc_hand_built_bank():
    """test_cp.cpp:110-134."""
    bank = np.array([0, 0, 0, 0, 2, -1, 0.5, 3], dtype=float).reshape(2, 4, 1)
    full = np.array([[0b1111]], dtype=np.uint64)
    out, pop = oracle.hsmc_extend_batch(bank, full, [0, 1], [1], [0, 0], np.zeros((0, 1)), [])
    assert pop[0] == 4
    out, pop = oracle.hsmc_extend_batch(bank, full, [0, 1], [1], [0, 1], [[1.0]], [1.0])
    assert pop[0] == 2 and int(out[0, 0]) == 0b0110
    with pytest.raises(IndexError):
        oracle.hsmc_extend_batch(bank, full, [0, 1], [2], [0, 1], [[1.0]], [1.0])


def test_hsmc_monotone_and_prefix_consistent():
    """test_cp.cpp:136-157."""
    cl = scalar_loop(0.9, 0.04, 0.04)
    bank = oracle.presample_bank(cl, 12, 256, 3)
    steps = [(t, (1.0, 0.35) if t % 2 else (-1.0, 0.5)) for t in range(1, 13)]
    m = np.full((1, 4), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    prev = 0.0
    for t, (a, b) in steps:
        m, pop = oracle.hsmc_extend_batch(bank, m, [0, 1], [t], [0, 1], [[a]], [b])
        cp = 1.0 - pop[0] / 256
        assert cp >= prev
        prev = cp
    full = np.full((1, 4), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    whole, pop = oracle.hsmc_extend_batch(bank, full, [0, 12], [t for t, _ in steps], np.arange(13),
                                          [[a] for _, (a, _) in steps], [b for _, (_, b) in steps])
    assert 1.0 - pop[0] / 256 == prev > 0.0
    assert np.array_equal(whole, m)


def test_mc_deterministic_cases():
    """test_cp.cpp:159-171."""
    cl = scalar_loop(1.0, 0.0, 0.0, w=0.0)
    w = {"bounds_lo": [-10.0], "bounds_hi": [10.0], "obs_lo": [[5.0]], "obs_hi": [[6.0]]}
    assert oracle.mc_certify(cl, w, [[0.0], [1.0], [2.0]], 100, 1, 0.01) == 0.0
    assert oracle.mc_certify(cl, w, [[0.0], [5.5]], 100, 1, 0.01) == 1.0
    with pytest.raises(ValueError):
        oracle.mc_certify(cl, w, [[0.0]], 0, 1, 0.01)


def test_mc_gaussian_tail_workers_seeds():
    """test_cp.cpp:173-192."""
    cl = scalar_loop(1.0, 0.0, 1.0)
    w = {"bounds_lo": [-1000.0], "bounds_hi": [1000.0], "obs_lo": [[1.6449]], "obs_hi": [[1000.0]]}
    n = 20000
    e1 = oracle.mc_certify(cl, w, [[0.0]], n, 11, 0.01)
    assert abs(e1 - 0.05) < 3 * math.sqrt(0.05 * 0.95 / n)
    assert oracle.mc_certify(cl, w, [[0.0]], n, 11, 0.01, workers=3) == e1
    e2 = oracle.mc_certify(cl, w, [[0.0]], n, 12, 0.01)
    pb = 0.5 * (e1 + e2)
    assert abs(e1 - e2) < 2.58 * math.sqrt(2 * pb * (1 - pb) / n)


# ------------------------------------------------------------ planning
def random_nodes(seed, n, obstacles, lo=-9.0, span=18.0, init=(-8.0, -8.0)):
    """test_plan.cpp:58-78."""
    w = box_world(obstacles)
    pos, vel = [list(init)], [[0.0, 0.0]]
    for i in range(n):
        p = [span * oracle.uniform(seed, i, 0, 0) + lo, span * oracle.uniform(seed, i, 0, 1) + lo]
        v = [2 * oracle.uniform(seed, i, 1, 0) - 1, 2 * oracle.uniform(seed, i, 1, 1) - 1]
        if not oracle.point_free(w, p):
            continue
        pos.append(p)
        vel.append(v)
    return np.array(pos), np.array(vel), w


def dijkstra(g):
    n = g["n_nodes"]
    dist = [math.inf] * n
    dist[0] = 0.0
    pq = [(0.0, 0)]
    while pq:
        d, v = heapq.heappop(pq)
        if d > dist[v]:
            continue
        for e in range(g["row_ptr"][v], g["row_ptr"][v + 1]):
            nd = d + g["edge_cost"][e]
            u = g["edge_to"][e]
            if nd < dist[u]:
                dist[u] = nd
                heapq.heappush(pq, (nd, u))
    return min([dist[v] for v in g["goal_nodes"]], default=math.inf)


def zero_bank(horizon, n, dw=2):
    return np.zeros((horizon + 1, n, dw))


def test_build_graph_degenerate_complete_and_parallel():
    """test_plan.cpp:82-122."""
    w = box_world([])
    goal = {"lo": [100.0, 100.0], "hi": [101.0, 101.0], "max_speed": 0.0}
    pos, vel = np.array([[0.0, 0], [5, 0], [9, 0]]), np.zeros((3, 2))
    assert oracle.build_graph(pos, vel, w, goal, 1e-6, 0.1, 0.05, 200.0).export()["n_edges"] == 0
    g = oracle.build_graph(pos, vel, w, goal, 1e6, 0.1, 0.05, 200.0).export()
    assert g["n_edges"] == 6
    goal2 = {"lo": [6.0, 6.0], "hi": [9.0, 9.0], "max_speed": 0.5}
    for seed in range(100, 110):
        pos, vel, w2 = random_nodes(seed, 30, [([-3, -3], [-1, 3]), ([1, -5], [3, 1])])
        a = oracle.build_graph(pos, vel, w2, goal2, 8.0, 0.25, 0.05, 200.0, workers=1).export()
        b = oracle.build_graph(pos, vel, w2, goal2, 8.0, 0.25, 0.05, 200.0, workers=4).export()
        assert np.array_equal(a["edge_to"], b["edge_to"])
        assert np.array_equal(a["edge_cost"], b["edge_cost"])


def test_explore_zero_noise_equals_dijkstra():
    """test_plan.cpp:131-158 and acceptance.cpp:179-253 (criterion 3)."""
    goal = {"lo": [5.0, 5.0], "hi": [9.0, 9.0], "max_speed": 0.6}
    solved = 0
    for seed in range(200, 206):
        pos, vel, w = random_nodes(seed, 60, [([-2, -6], [0, 4])])
        gh = oracle.build_graph(pos, vel, w, goal, 9.0, 0.25, 0.05, 200.0, workers=W)
        g = gh.export()
        res = oracle.explore(gh, zero_bank(4096, 8), 0.25, 1.0, 0.5, 9.0, workers=W, masks=False)
        best = min([res["cost"][i] for i in res["goal_plans"]], default=math.inf)
        ref = dijkstra(g)
        assert best == ref
        solved += not math.isinf(ref)
    assert solved >= 3


def test_explore_trivial_and_disconnected():
    """test_plan.cpp:160-186."""
    w = box_world([])
    pos, vel = np.array([[0.0, 0.0], [5.0, 5.0]]), np.zeros((2, 2))
    g = oracle.build_graph(pos, vel, w, {"lo": [-1, -1], "hi": [1, 1], "max_speed": 0.1}, 1e6, 0.25, 0.05, 200.0)
    r = oracle.explore(g, zero_bank(64, 8), 0.5, 1.0, 0.5, 1e6)
    assert r["termination"] == "goal_below_alpha_min" and r["cost"][r["goal_plans"][0]] == 0.0
    g2 = oracle.build_graph(pos, vel, w, {"lo": [100, 100], "hi": [101, 101], "max_speed": 0.0}, 1e6, 0.25, 0.05,
                            200.0)
    r2 = oracle.explore(g2, zero_bank(64, 8), 0.5, 1.0, 0.5, 1e6)
    assert len(r2["goal_plans"]) == 0 and r2["termination"] == "frontier_exhausted"


def noisy_setup(seed=777, n=80):
    scn = {"workspace": {"bounds": {"lo": [-10, -10], "hi": [10, 10]},
                         "obstacles": [{"lo": [-1, -4], "hi": [1, 6]}]},
           "start": {"position": [-8, -8]}, "goal": {"lo": [5, 5], "hi": [9, 9], "max_speed": 0.6},
           "noise": {"process": [0, 0, 0.02, 0.02], "measurement": 0.01, "initial": 0.005},
           "dt": 0.25, "samples": 10, "alpha": 0.05}
    cl, _ = oracle.scenario_models(json.dumps(scn))
    pos, vel, w = random_nodes(seed, n, [([-1, -4], [1, 6])])
    g = oracle.build_graph(pos, vel, w, {"lo": [5, 5], "hi": [9, 9], "max_speed": 0.6}, 9.0, 0.25, 0.05, 200.0,
                           workers=W)
    return cl, g


def test_explore_identical_across_workers():
    """test_plan.cpp:188-227 and acceptance.cpp:435-471 (criterion 8 identity)."""
    cl, g = noisy_setup()
    bank = oracle.presample_bank(cl, 2048, 64, 9, workers=W)
    r1 = oracle.explore(g, bank, 0.01, 0.2, 0.5, 9.0, workers=1)
    r8 = oracle.explore(g, bank, 0.01, 0.2, 0.5, 9.0, workers=8)
    for k in ("head", "parent", "cost", "cp_hat", "masks", "goal_plans"):
        assert np.array_equal(r1[k], r8[k]), k
    assert r1["partial_plans"] == r8["partial_plans"]


def test_explore_pareto_invariants():
    """acceptance.cpp:475-571 (criterion 9) on a sample of the mini scenarios."""
    base = {"workspace": {"bounds": {"lo": [-5, -5], "hi": [5, 5]}}, "start": {"position": [-4.5, -4.5]},
            "goal": {"lo": [3, 3], "hi": [4.8, 4.8], "max_speed": 0.8}, "dt": 0.25, "samples": 5, "alpha": 0.05}
    run = 0
    for trial in range(0, 1000, 25):
        obs = []
        for i in range(int(3 * oracle.uniform(trial, 50, 0, 0))):
            cx, cy = 6 * oracle.uniform(trial, 51, i, 0) - 3, 6 * oracle.uniform(trial, 51, i, 1) - 3
            wx, wy = 0.4 + oracle.uniform(trial, 51, i, 2), 0.4 + oracle.uniform(trial, 51, i, 3)
            obs.append(([cx - wx, cy - wy], [cx + wx, cy + wy]))
        w = {"bounds_lo": [-5.0, -5.0], "bounds_hi": [5.0, 5.0], "obs_lo": [o[0] for o in obs],
             "obs_hi": [o[1] for o in obs]}
        if not oracle.point_free(w, [-4.5, -4.5]):
            continue
        q = 0.002 + 0.02 * oracle.uniform(trial, 52, 0, 0)
        scn = dict(base, noise={"process": [0, 0, q, q], "measurement": 0.01, "initial": 0.002},
                   workspace={"bounds": base["workspace"]["bounds"],
                              "obstacles": [{"lo": o[0], "hi": o[1]} for o in obs]})
        cl, _ = oracle.scenario_models(json.dumps(scn))
        pos, vel = [[-4.5, -4.5]], [[0.0, 0.0]]
        for i in range(12):
            p = [9.6 * oracle.uniform(trial, 53, i, 0) - 4.8, 9.6 * oracle.uniform(trial, 53, i, 1) - 4.8]
            v = [1.6 * oracle.uniform(trial, 54, i, 0) - 0.8, 1.6 * oracle.uniform(trial, 54, i, 1) - 0.8]
            if oracle.point_free(w, p):
                pos.append(p)
                vel.append(v)
        try:
            g = oracle.build_graph(np.array(pos), np.array(vel), w, {"lo": [3, 3], "hi": [4.8, 4.8],
                                                                     "max_speed": 0.8}, 7.0, 0.25, 0.05, 100.0)
        except RuntimeError:
            continue
        bank = oracle.presample_bank(cl, 512, 32, trial + 1)
        amax = 0.05 + 0.3 * oracle.uniform(trial, 55, 0, 0)
        inv = oracle.explore_invariants(g, bank, amax / 4, amax, 0.5, 7.0)
        assert inv["dominance"] == 0 and inv["double_expansions"] == 0 and inv["cp"] == 0
        run += 1
    assert run >= 30


def test_bisect_select_traces():
    """test_plan.cpp:229-248."""
    s = oracle.bisect_select([0.004, 0.02, 0.08], 0.05)
    assert s["success"] and s["plan_id"] == 1 and s["mc"] == 0.02
    assert not oracle.bisect_select([0.2, 0.4], 0.05)["success"]
    s = oracle.bisect_select([0.01], 0.05)
    assert s["success"] and s["plan_id"] == 0
    assert not oracle.bisect_select([], 0.05)["success"]


def test_run_pump_deterministic_and_constrained():
    """test_plan.cpp:311-346 on the bundled minimal scenario."""
    txt = scenario_text("minimal")
    j = json.loads(txt)
    j["mc_samples"] = 2000
    txt = json.dumps(j)
    r1 = oracle.run_pump(txt, workers=1)
    r4 = oracle.run_pump(txt, workers=4)
    for k in ("success", "cost", "certified_cp", "partial_plans"):
        assert r1[k] == r4[k]
    assert np.array_equal(r1["path"], r4["path"])
    assert r1["success"] and r1["certified_cp"] <= j["alpha"] and r1["cp_hat"] < 2 * j["alpha"]


def test_glibc_and_portable_normals_give_the_same_decisions():
    """The bank bits differ between glibc and portable normals, but every
    HSMC kill decision and hence the whole exploration is unchanged."""
    cl, g = noisy_setup(seed=778, n=60)
    oracle.set_normal_mode(oracle.GLIBC)
    bg = oracle.presample_bank(cl, 1024, 64, 9, workers=W)
    oracle.set_normal_mode(oracle.PORTABLE)
    bp = oracle.presample_bank(cl, 1024, 64, 9, workers=W)
    assert not np.array_equal(bg.view(np.uint64), bp.view(np.uint64))  # bits differ
    rg = oracle.explore(g, bg, 0.01, 0.2, 0.5, 9.0, workers=W)
    rp = oracle.explore(g, bp, 0.01, 0.2, 0.5, 9.0, workers=W)
    for k in ("head", "parent", "cost", "cp_hat", "masks", "goal_plans"):
        assert np.array_equal(rg[k], rp[k]), k


def test_repeated_rrt_kat(oracle_lib):
    """test_plan.cpp:279-306: empty workspace succeeds (cost above the direct
    connection to the reached end state), sealed goal fails."""
    import json as _json

    base = {"name": "rrt_kat", "workspace": {"bounds": {"lo": [-10, -10], "hi": [10, 10]}, "obstacles": []},
            "start": {"position": [-5, 0], "velocity": [0, 0]},
            "goal": {"lo": [4, -1], "hi": [6, 1], "max_speed": 0.5},
            "noise": {"process": [0, 0, 0, 0], "measurement": 0, "initial": 0},
            "dt": 0.25, "alpha": 0.05, "max_speed": 1.0, "connection_radius": 6.0, "mc_samples": 200,
            "rrt": {"max_iterations": 80}, "samples": 10}
    ok = oracle_lib.repeated_rrt(_json.dumps(base), 40, 0.05, 200, workers=4)
    assert ok["success"] and len(ok["traj_t"]) > 0
    end_p, end_v = ok["traj_pos"][-1], ok["traj_vel"][-1]
    direct = oracle_lib.connect([-5, 0], [0, 0], end_p, end_v, 200.0)
    assert ok["cost"] >= direct["cost"] - 1e-6
    sealed = dict(base)
    sealed["workspace"] = {"bounds": {"lo": [-10, -10], "hi": [10, 10]}, "obstacles": [{"lo": [3, -3], "hi": [7, 3]}]}
    fail = oracle_lib.repeated_rrt(_json.dumps(sealed), 20, 0.05, 200, workers=4)
    assert not fail["success"]
