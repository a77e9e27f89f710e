"""Parity at the full BASELINE configs (north_star: "bit-exact Pareto set and
selected plan versus the CPU reference"), through the C ABI, at the sizes
bench.py measures: configs[0] quad3d_three_obstacle (n = 2000, 32 particles),
configs[1] quad3d_indoor (n = 4000, 64 particles), configs[2] quad3d_forest
(n = 16000, 128 particles, 200 boxes), each with its full 20000 MC rollouts.

Per config: the graph (every edge, waypoint and half-space, by bit
pattern), the explore arena (every record, mask, Pareto set, goal plan and
statistic: planner.hpp:264-265) and the whole solve (front, MC probe trace,
selected plan, smoothing, trajectory bits: pump.hpp:170-263).  At these sizes
the pipelined rounds, the > 1024-member dominance pass and the MC-table
growth all run.  The oracle takes ~1, 3 and 40 s on 16 host threads."""
import json
import os

import pytest

from conftest import scenario_text
from test_gpu_planner import assert_graph_equal, assert_run_equal, explore_equal, goal_of, ws_of

pytestmark = pytest.mark.gpu

WORKERS = max(1, min(32, os.cpu_count() or 4))


@pytest.mark.parametrize("name", ["quad3d_three_obstacle", "quad3d_indoor", "quad3d_forest"])
def test_named_config_full_size(oracle_lib, gpu_ctx, name):
    from paper_1607_06886_b200 import api

    txt = scenario_text(name)
    j = json.loads(txt)
    cl, sc = oracle_lib.scenario_models(txt)
    pos, vel = oracle_lib.scenario_nodes(txt)
    args = (ws_of(j), goal_of(j), sc["r_n"], sc["dt"], sc["eps_cc"], sc["tau_max"])
    og = oracle_lib.build_graph(pos, vel, *args, workers=WORKERS)
    gg = api.build_graph(pos, vel, *args, ctx=gpu_ctx)
    assert_graph_equal(gg.export(), og.export())
    # explore arena on the scenario's own bank
    bank = api.presample_bank(cl, j["bank_horizon"], j["particles"], j["seeds"]["bank"], ctx=gpu_ctx)
    eta = sc["eta"]
    amin, amax = sc["alpha"] / eta, min(1.0, eta * sc["alpha"])
    ref_x = oracle_lib.explore(og, bank, amin, amax, sc["lambda"], sc["r_n"], workers=WORKERS)
    got_x = api.explore(gg, amin, amax, sc["lambda"], sc["r_n"], ctx=gpu_ctx)
    explore_equal(got_x, ref_x)
    assert ref_x["partial_plans"] > 1e5 if name == "quad3d_forest" else ref_x["partial_plans"] > 1e4
    # the whole solve, full MC
    got = api.run_pump(api.parse_scenario(txt), ctx=gpu_ctx)
    ref = oracle_lib.run_pump(txt, workers=WORKERS, prebuilt=og)
    assert_run_equal(got, ref)
    assert got["success"] == 1 and got["partial_plans"] == ref_x["partial_plans"]
