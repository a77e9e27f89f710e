"""Subprocess helper for tests/test_gpu_kernels.py::test_mc_kernel_paths: the
MC certification parity cases (axis-separable and coupled closed loops) under
a PUMP_MC_* environment (the kernel path is fixed per process).  Prints "ok"
on success."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
from conftest import coupled_noise_text, scenario_text  # noqa: E402
from paper_1607_06886_b200 import api  # noqa: E402

ctx = api.Context(0)
for name, n_mc in [("quad3d_three_obstacle", 3000), ("three_obstacle", 2000), ("coupled", 2000)]:
    txt = coupled_noise_text() if name == "coupled" else scenario_text(name)
    cl, sc = oracle.scenario_models(txt)
    j = json.loads(txt)
    dw = cl["dw"]
    ws = {"bounds_lo": j["workspace"]["bounds"]["lo"], "bounds_hi": j["workspace"]["bounds"]["hi"],
          "obs_lo": [o["lo"] for o in j["workspace"]["obstacles"]],
          "obs_hi": [o["hi"] for o in j["workspace"]["obstacles"]]}
    start = np.array(j["start"]["position"], float)
    goal = 0.5 * (np.array(j["goal"]["lo"], float) + np.array(j["goal"]["hi"], float))
    ts = np.linspace(0, 1, 120)[:, None]
    y = start + ts * (goal - start)
    y[:, 1 % dw] += 0.3 * np.sin(np.pi * ts[:, 0])
    y = np.clip(y, np.array(ws["bounds_lo"]) + 0.01, np.array(ws["bounds_hi"]) - 0.01)
    for traj in (y, y[:40]):
        got = int(api.mc_certify_batch(cl, ws, [traj], 0, n_mc, 2, sc["eps_cc"], ctx)[0])
        ref = oracle.mc_hits(cl, ws, traj, 0, n_mc, 2, sc["eps_cc"], workers=8)
        assert got == ref, (name, got, ref)
print("ok")
