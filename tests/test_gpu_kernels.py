"""GPU parity of the particle bank (K_bank), batched HSMC (K_hsmc) and MC
certification (K_mc) against the CPU oracle, through the C ABI.

Bar: bit-exact (bank doubles compared by their bit patterns, masks word for
word, hit counts and per-rollout flags exactly).
"""
import json
import os

import numpy as np
import pytest

from conftest import scenario_text

pytestmark = pytest.mark.gpu


def scalar_loop(a, v, s0, w=1.0):
    """test_cp.cpp:13-31 ScalarSetup closed loop (L = K = 0): F = diag(a, a)."""
    return {"d": 1, "dw": 1, "F": np.array([[a, 0.0], [0.0, a]]), "Gv": np.array([[1.0], [0.0]]),
            "Gw": np.array([[0.0], [0.0]]), "Sv": np.array([[np.sqrt(v)]]), "Sw": np.array([[np.sqrt(w)]]),
            "S0": np.array([[np.sqrt(s0)]]), "C": np.array([[1.0]])}


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


@pytest.mark.parametrize("name,T,n", [("minimal", 64, 512), ("three_obstacle", 300, 96),
                                      ("quad3d_three_obstacle", 512, 32), ("quad3d_indoor", 257, 64)])
def test_bank_bit_exact(oracle_lib, gpu_ctx, name, T, n):
    from paper_1607_06886_b200 import api

    cl, _ = oracle_lib.scenario_models(scenario_text(name))
    ref = oracle_lib.presample_bank(cl, T, n, 7, workers=8)
    got = api.presample_bank(cl, T, n, 7, ctx=gpu_ctx)
    assert got.shape == ref.shape
    assert np.array_equal(bits(got), bits(ref))


def test_bank_scalar_and_zero_noise(oracle_lib, gpu_ctx):
    from paper_1607_06886_b200 import api

    cl = scalar_loop(0.9, 0.04, 0.04)
    ref = oracle_lib.presample_bank(cl, 12, 256, 3)
    got = api.presample_bank(cl, 12, 256, 3, ctx=gpu_ctx)
    assert np.array_equal(bits(got), bits(ref))
    z = scalar_loop(1.0, 0.0, 0.0, w=0.0)
    assert np.all(api.presample_bank(z, 10, 16, 7, ctx=gpu_ctx) == 0.0)  # test_lti.cpp:185-195


def test_hsmc_hand_built_kat(gpu_ctx):
    """test_cp.cpp:110-134."""
    from paper_1607_06886_b200 import api

    bank = np.array([0, 0, 0, 0, 2, -1, 0.5, 3], dtype=float).reshape(2, 4, 1)
    api.bank_upload(bank, gpu_ctx)
    full = api.full_mask(4)
    m, cp = api.hsmc_extend(full, [(1, None)], 4, gpu_ctx)
    assert cp == 0.0 and np.array_equal(m, full)
    m, cp = api.hsmc_extend(full, [(1, [([1.0], 1.0)])], 4, gpu_ctx)
    assert cp == 0.5
    assert int(m[0]) == 0b0110
    with pytest.raises(IndexError):
        api.hsmc_extend(full, [(2, [([1.0], 1.0)])], 4, gpu_ctx)
    with pytest.raises(IndexError):  # range check precedes the null-region skip
        api.hsmc_extend(full, [(2, None)], 4, gpu_ctx)


@pytest.mark.parametrize("name,n", [("quad3d_three_obstacle", 32), ("quad3d_indoor", 64), ("three_obstacle", 512),
                                    ("quad3d_three_obstacle", 100)])
def test_hsmc_random_tasks(oracle_lib, gpu_ctx, name, n):
    from paper_1607_06886_b200 import api

    rng = np.random.default_rng(5)
    cl, _ = oracle_lib.scenario_models(scenario_text(name))
    T = 200
    bank = api.presample_bank(cl, T, n, 11, ctx=gpu_ctx)
    dw = cl["dw"]
    n_tasks = 3000
    W = (n + 63) // 64
    masks = rng.integers(0, 2 ** 63, size=(n_tasks, W), dtype=np.int64).astype(np.uint64)
    masks &= api.full_mask(n)[None, :]
    masks[::3] = api.full_mask(n)
    nst = rng.integers(0, 25, size=n_tasks)
    step_off = np.concatenate([[0], np.cumsum(nst)]).astype(np.int64)
    S = int(step_off[-1])
    step_t = rng.integers(0, T + 1, size=S).astype(np.int32)
    nh = rng.integers(0, 4, size=S)
    hs_off = np.concatenate([[0], np.cumsum(nh)]).astype(np.int64)
    H = int(hs_off[-1])
    sd = float(np.std(bank))
    hs_a = rng.normal(size=(H, dw))
    hs_b = rng.normal(scale=2 * sd, size=H) + 0.5 * sd
    ref_m, ref_p = oracle_lib.hsmc_extend_batch(bank, masks, step_off, step_t, hs_off, hs_a, hs_b, workers=8)
    got_m, got_p = api.hsmc_extend_batch(masks, step_off, step_t, hs_off, hs_a, hs_b, gpu_ctx)
    assert np.array_equal(got_m, ref_m)
    assert np.array_equal(got_p, ref_p)
    assert 0 < ref_p.sum() < n * n_tasks  # nontrivial kills


def test_mc_deterministic_cases(gpu_ctx):
    """test_cp.cpp:159-171."""
    from paper_1607_06886_b200 import api

    cl = scalar_loop(1.0, 0.0, 0.0, w=0.0)
    ws = {"bounds_lo": [-10.0], "bounds_hi": [10.0], "obs_lo": [[5.0]], "obs_hi": [[6.0]]}
    assert api.mc_certify([[0.0], [1.0], [2.0]], cl, ws, 100, 1, 0.01, gpu_ctx) == 0.0
    assert api.mc_certify([[0.0], [5.5]], cl, ws, 100, 1, 0.01, gpu_ctx) == 1.0
    with pytest.raises(ValueError):
        api.mc_certify([], cl, ws, 100, 1, 0.01, gpu_ctx)


def test_mc_gaussian_tail(oracle_lib, gpu_ctx):
    """test_cp.cpp:173-192: N(0,1) position, obstacle x >= 1.6449 -> 5%."""
    from paper_1607_06886_b200 import api

    cl = scalar_loop(1.0, 0.0, 1.0)
    ws = {"bounds_lo": [-1000.0], "bounds_hi": [1000.0], "obs_lo": [[1.6449]], "obs_hi": [[1000.0]]}
    n = 20000
    v1 = api.mc_certify([[0.0]], cl, ws, n, 11, 0.01, gpu_ctx)
    assert abs(v1 - 0.05) < 3 * np.sqrt(0.05 * 0.95 / n)
    assert v1 == oracle_lib.mc_certify(cl, ws, [[0.0]], n, 11, 0.01, workers=8)
    # shards add up exactly (multi-GPU split invariance)
    h = sum(int(api.mc_certify_batch(cl, ws, [[[0.0]]], lo, hi, 11, 0.01, gpu_ctx)[0])
            for lo, hi in [(0, 7000), (7000, 7001), (7001, 20000)])
    assert h == round(v1 * n)


@pytest.mark.parametrize("name,n_mc", [("quad3d_three_obstacle", 4000), ("three_obstacle", 3000),
                                       ("quad3d_indoor", 3000)])
def test_mc_trajectories_match_oracle(oracle_lib, gpu_ctx, name, n_mc):
    """Real trajectories near obstacles: per-rollout flags must agree."""
    from paper_1607_06886_b200 import api

    txt = scenario_text(name)
    cl, sc = oracle_lib.scenario_models(txt)
    j = json.loads(txt)
    dw = cl["dw"]
    ws = {"bounds_lo": j["workspace"]["bounds"]["lo"], "bounds_hi": j["workspace"]["bounds"]["hi"],
          "obs_lo": [o["lo"] for o in j["workspace"]["obstacles"]],
          "obs_hi": [o["hi"] for o in j["workspace"]["obstacles"]]}
    # straight line start -> goal centre grazing the first obstacle corner region
    start = np.array(j["start"]["position"], float)
    goal = 0.5 * (np.array(j["goal"]["lo"], float) + np.array(j["goal"]["hi"], float))
    ts = np.linspace(0, 1, 120)[:, None]
    y = start + ts * (goal - start)
    y[:, 1 % dw] += 0.3 * np.sin(np.pi * ts[:, 0])
    # keep the nominal itself free: clip into bounds
    y = np.clip(y, np.array(ws["bounds_lo"]) + 0.01, np.array(ws["bounds_hi"]) - 0.01)
    ref_hits, ref_flags = oracle_lib.mc_hits(cl, ws, y, 0, n_mc, 2, sc["eps_cc"], workers=8, want_flags=True)
    got = api.mc_certify_batch(cl, ws, [y, y[:40]], 0, n_mc, 2, sc["eps_cc"], gpu_ctx)
    assert int(got[0]) == ref_hits
    ref40 = oracle_lib.mc_hits(cl, ws, y[:40], 0, n_mc, 2, sc["eps_cc"], workers=8)
    assert int(got[1]) == ref40
    # per-rollout flags via one-rollout shards on a sample
    idx = np.flatnonzero(ref_flags)[:20].tolist() + list(range(20))
    for i in idx:
        h = int(api.mc_certify_batch(cl, ws, [y], i, i + 1, 2, sc["eps_cc"], gpu_ctx)[0])
        assert h == int(ref_flags[i])


@pytest.mark.parametrize("env", [{}, {"PUMP_MC_DIRECT": "1"}])
def test_mc_kernel_paths(env):
    """Every MC kernel path stays bit-exact: the common-random-number table
    (separable and dense builds), and the direct kernels used when the table
    would not fit in memory (PUMP_MC_DIRECT: lane-per-axis and dense), on
    separable and coupled closed loops."""
    import subprocess
    import sys

    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "mc_paths_check.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
