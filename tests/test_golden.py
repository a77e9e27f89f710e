"""Golden fixtures (tests/golden/golden.json, made by make_golden.py).

CPU: the oracle reproduces them.  GPU: the library reproduces them on the
B200 without consulting the oracle at run time.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, scenario_text

with open(os.path.join(GOLDEN, "golden.json")) as f:
    G = json.load(f)


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def variant(name, kw):
    j = json.loads(scenario_text(name))
    j.update(kw)
    return json.dumps(j)


def check_run(r, g):
    assert int(r["success"]) == g["success"]
    assert r["path"].tolist() == g["path"]
    assert int(np.float64(r["cost"]).view(np.uint64)) == g["cost_bits"]
    assert r["certified_cp"] == g["certified_cp"] and r["cp_hat"] == g["cp_hat"]
    assert r["partial_plans"] == g["partial_plans"] and r["termination"] == g["termination"]
    assert r["mc_eval_ids"].tolist() == g["mc_eval_ids"] and r["mc_eval_values"].tolist() == g["mc_eval_values"]
    assert r["pareto_cp"].tolist() == g["pareto_cp"] and r["smoothing_s"] == g["smoothing_s"]
    assert digest(r["traj_t"], r["traj_pos"], r["traj_vel"], r["traj_ctrl"]) == g["traj_sha256"]


def test_oracle_normals_golden(oracle_lib):
    keys = np.arange(256, dtype=np.uint64)
    oracle_lib.set_normal_mode(oracle_lib.PORTABLE)
    assert oracle_lib.normals(1, keys, 0, 0).view(np.uint64).tolist() == G["normals_seed1_portable_bits"]


def test_oracle_banks_golden(oracle_lib):
    for name, g in G["banks"].items():
        cl, _ = oracle_lib.scenario_models(scenario_text(name))
        b = oracle_lib.presample_bank(cl, g["T"], g["n"], g["seed"], workers=4)
        assert digest(b) == g["sha256"], name


@pytest.mark.parametrize("name", list(G["runs"]))
def test_oracle_runs_golden(oracle_lib, name):
    g = G["runs"][name]
    check_run(oracle_lib.run_pump(variant(name, g["overrides"]), workers=os.cpu_count() or 4), g)


@pytest.mark.gpu
def test_gpu_banks_golden(gpu_ctx):
    from paper_1607_06886_b200 import api

    for name, g in G["banks"].items():
        cl = api.parse_scenario(scenario_text(name)).closed_loop()
        b = api.presample_bank(cl, g["T"], g["n"], g["seed"], ctx=gpu_ctx)
        assert digest(b) == g["sha256"], name


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(G["runs"]))
def test_gpu_runs_golden(gpu_ctx, name):
    from paper_1607_06886_b200 import api

    g = G["runs"][name]
    check_run(api.run_pump(api.parse_scenario(variant(name, g["overrides"])), ctx=gpu_ctx), g)
