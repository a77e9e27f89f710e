import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SCENARIOS = "/root/reference/proj/scenarios"  # only read when present (never on the GPU box)
SCENARIOS = os.path.join(ROOT, "scenarios")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    oracle.build()
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_1607_06886_b200 import api

    ctx = api.Context(0)
    yield ctx
    ctx.close()


def scenario_text(name: str) -> str:
    """2-D reference scenarios are committed as golden copies under
    tests/golden/scenarios (the GPU box has no /root/reference); 3-D ones live
    in scenarios/."""
    for d in (os.path.join(GOLDEN, "scenarios"), SCENARIOS):
        p = os.path.join(d, name + ".json")
        if os.path.exists(p):
            with open(p) as f:
                return f.read()
    raise FileNotFoundError(name)


def coupled_noise_text(samples=500, mc=3000):
    """quad3d_three_obstacle with full-matrix (cross-axis correlated) process
    and measurement noise and a coupled tracking weight: the closed loop is
    not axis-separable, so the dense bank (k_bank_rec<6,3>) and dense MC-table
    (k_mctab_dense) kernels run (scenario.hpp:110 accepts full matrices)."""
    import json

    import numpy as np

    j = json.loads(scenario_text("quad3d_three_obstacle"))
    q = np.diag([0.0, 0.0, 0.0, 3e-4, 3e-4, 3e-4])
    q[3, 4] = q[4, 3] = 1e-4
    q[4, 5] = q[5, 4] = -0.5e-4
    q[0, 3] = q[3, 0] = 1e-6
    q[0, 0] = 1e-5
    w = np.diag([5e-4, 5e-4, 5e-4])
    w[0, 1] = w[1, 0] = 2e-4
    Q = np.eye(6)
    Q[0, 1] = Q[1, 0] = 0.3
    j["noise"]["process"] = q.tolist()
    j["noise"]["measurement"] = w.tolist()
    j["tracking"] = {"Q": Q.tolist()}
    j["samples"] = samples
    j["mc_samples"] = mc
    return json.dumps(j)
