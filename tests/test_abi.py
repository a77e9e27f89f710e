"""The C-ABI library (CPU-side checks, no GPU needed).

- libpump_gpu.so loads and exports every function include/pump_gpu.h declares;
- without a B200 the library fails loudly (PUMP_E_CUDA), never falls back;
- scenario parsing / validation errors follow scenario.hpp:144-257 and map to
  the reference's exception types (ScenarioError, exit code 1 in the CLI).
"""
import ctypes as C
import json
import os
import re

import pytest

from conftest import ROOT, scenario_text


def declared_functions():
    with open(os.path.join(ROOT, "include", "pump_gpu.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|double|int64_t|char\s*\*|const char\s*\*|void)\s*\*?\s*(pump_\w+)\s*\(",
                       text, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_1607_06886_b200 import api

    L = api.lib()
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(api.EXPORTS) <= set(names)
    assert L.pump_abi_version() == 1


def test_oracle_is_a_separate_library():
    """The product never links the oracle (test infrastructure)."""
    from paper_1607_06886_b200 import api

    with open(api.LIB_PATH, "rb") as f:
        blob = f.read()
    assert b"oracle_" not in blob and b"liboracle" not in blob


def test_no_gpu_fails_loudly():
    import torch

    from paper_1607_06886_b200 import api

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(api.PumpCudaError):
        api.Context(0)


def test_scenario_validation_messages():
    from paper_1607_06886_b200 import api

    with pytest.raises(api.ScenarioError, match="missing required key"):
        api.parse_scenario(json.dumps({"alpha": 2}))
    j = json.loads(scenario_text("minimal"))
    j["bogus"] = 1
    with pytest.raises(api.ScenarioError, match='unknown key "bogus"'):
        api.parse_scenario(json.dumps(j))
    j = json.loads(scenario_text("minimal"))
    j["alpha"] = 1.5
    with pytest.raises(api.ScenarioError, match="alpha"):
        api.parse_scenario(json.dumps(j))
    j = json.loads(scenario_text("minimal"))
    j["start"]["position"] = [5.0, 2.0]  # inside the obstacle
    with pytest.raises(api.ScenarioError, match="collision"):
        api.parse_scenario(json.dumps(j))
    with pytest.raises(api.ScenarioError, match="cannot open"):
        api.load_scenario("/nonexistent/scenario.json")
    with pytest.raises(api.ScenarioError, match="parse error"):
        api.parse_scenario("{not json")


def test_scenario_derived_parameters_and_models_match_oracle(oracle_lib):
    """Derived quantities (scenario.hpp:63-75, graph.hpp:41-48) and the
    closed-loop matrices are computed by the same host code on both sides."""
    import numpy as np

    from paper_1607_06886_b200 import api

    for name in ("minimal", "indoor", "quad3d_three_obstacle", "quad3d_indoor"):
        txt = scenario_text(name)
        s = api.parse_scenario(txt)
        p = s.params()
        cl = s.closed_loop()
        ocl, osc = oracle_lib.scenario_models(txt)
        for k in ("eps_cc", "r_n", "tau_max", "alpha", "eta", "lambda", "dt"):
            assert p[k] == osc[k], k
        for k in ("F", "Gv", "Gw", "Sv", "Sw", "S0", "C"):
            assert np.array_equal(cl[k], ocl[k]), k
    # defaults: eta 2 above 1%, 10 below; eps_cc = min edge / 100
    j = json.loads(scenario_text("minimal"))
    j["alpha"] = 0.005
    del j["collision_resolution"]
    p = api.parse_scenario(json.dumps(j)).params()
    assert p["eta"] == 10.0
    assert p["eps_cc"] == 2.0 / 100.0  # min over bounds (10, 10) and the box (2, 5)


def test_closed_loop_is_stable_and_separable(oracle_lib):
    """The double-integrator LQG loop has spectral radius < 1 and the axis
    structure the separable MC kernel relies on."""
    import numpy as np

    cl, _ = oracle_lib.scenario_models(scenario_text("quad3d_indoor"))
    assert max(abs(np.linalg.eigvals(cl["F"]))) < 1.0
    d, dw = cl["d"], cl["dw"]
    ax = [(i % d) % dw for i in range(2 * d)]
    for r in range(2 * d):
        for c in range(2 * d):
            if ax[r] != ax[c]:
                assert cl["F"][r, c] == 0.0
