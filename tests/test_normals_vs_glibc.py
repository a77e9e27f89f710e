"""The literal reference draws its normals with glibc log / cos; the build
(kernels and oracle alike) with the correctly rounded pmath.h ones.  They
differ only where glibc is not correctly rounded (~0.15% of normals,
tests/test_pmath.py), by one ulp.  This measures what that does to a solve
at the full BASELINE configs: the oracle in GLIBC mode (the reference's
semantics; pinned to oracle/_ref by tests/test_ref_crosscheck.py) against
PORTABLE mode (what the GPU computes, bit for bit).

Decisions must be identical: particle-bank kill tests (every explore record
and mask), the Pareto front, the bisection's probe sequence, the selected
plan and the smoothing fraction.  Stated tolerance on certified CP values:
|delta| <= 2 / n_mc (at most two of the 20000 rollouts may flip).  Runs on the
GPU box's host cores (the oracle is CPU code; ~2 x 40 s for the forest)."""
import json
import os

import numpy as np
import pytest

from conftest import scenario_text

WORKERS = max(1, min(32, os.cpu_count() or 4))


def _bank_and_solve(oracle, txt, mode):
    oracle.set_normal_mode(mode)
    try:
        j = json.loads(txt)
        cl, _ = oracle.scenario_models(txt)
        bank = oracle.presample_bank(cl, j["bank_horizon"], j["particles"], j["seeds"]["bank"], workers=WORKERS)
        r = oracle.run_pump(txt, workers=WORKERS)
    finally:
        oracle.set_normal_mode(oracle.PORTABLE)
    return bank, r


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["quad3d_three_obstacle", "quad3d_indoor", "quad3d_forest"])
def test_glibc_and_portable_normals_full_size(oracle_lib, name):
    txt = scenario_text(name)
    bg, rg = _bank_and_solve(oracle_lib, txt, oracle_lib.GLIBC)
    bp, rp = _bank_and_solve(oracle_lib, txt, oracle_lib.PORTABLE)
    differ = int(np.count_nonzero(bg.view(np.uint64) != bp.view(np.uint64)))
    print(f"{name}: bank entries differing {differ} of {bg.size} ({100.0 * differ / bg.size:.4f}%); "
          f"certified CP glibc {rg['certified_cp']} portable {rp['certified_cp']}; mc evals "
          f"{list(zip(rg['mc_eval_ids'].tolist(), rg['mc_eval_values'].tolist()))} vs "
          f"{list(zip(rp['mc_eval_ids'].tolist(), rp['mc_eval_values'].tolist()))}")
    for k in ("success", "partial_plans", "termination", "path_len", "n_pareto", "n_mc_evals"):
        assert rg[k] == rp[k], (k, rg[k], rp[k])
    assert np.array_equal(rg["path"], rp["path"])
    assert np.array_equal(rg["pareto_cost"], rp["pareto_cost"])
    assert np.array_equal(rg["pareto_cp"], rp["pareto_cp"])
    assert np.array_equal(rg["mc_eval_ids"], rp["mc_eval_ids"])
    n_mc = json.loads(txt)["mc_samples"]
    assert np.all(np.abs(rg["mc_eval_values"] - rp["mc_eval_values"]) <= 2.0 / n_mc + 1e-15)
    assert rg["smoothing_s"] == rp["smoothing_s"]
    assert abs(rg["certified_cp"] - rp["certified_cp"]) <= 2.0 / n_mc + 1e-15
    assert rg["cost"] == rp["cost"]
