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
