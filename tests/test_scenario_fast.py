"""The strict fast scenario reader (csrc/host/scenario_fast.hpp) against the
nlohmann loader (csrc/host/scenario.hpp, the restatement of scenario.hpp):
on every bundled scenario and on mutations of them (missing / unknown /
duplicate keys, wrong types, floats for counts, escapes, invalid values) it
either builds the identical Scenario or defers to the loader; it never accepts
what the loader rejects."""
import glob
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1607_06886_b200", "csrc")
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("sfc") / "scenario_fast_check")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", CSRC, "-I", JSON_INC,
                    os.path.join(ROOT, "tools", "checks", "scenario_fast_check.cpp"), "-o", out], check=True)
    return out


def mutations(j):
    yield "same", j
    yield "pretty", j  # (written indented below)
    for k in list(j):
        if k not in ("name",):
            d = dict(j)
            del d[k]
            yield f"no_{k}", d
    yield "unknown_key", dict(j, zzz=1)
    yield "samples_float", dict(j, samples=float(j["samples"]))
    yield "samples_frac", dict(j, samples=j["samples"] + 0.5)
    yield "samples_str", dict(j, samples=str(j["samples"]))
    yield "samples_neg", dict(j, samples=-3)
    yield "samples_huge", dict(j, samples=2 ** 70)
    yield "dt_bool", dict(j, dt=True)
    yield "dt_int", dict(j, dt=1)
    yield "alpha_zero", dict(j, alpha=0)
    yield "alpha_exp", dict(j, alpha=5e-2)
    yield "name_num", dict(j, name=3)
    yield "name_unicode", dict(j, name="förest")
    yield "name_escape", dict(j, name="a\\tb")
    yield "seed_neg", dict(j, seeds={"bank": -1})
    yield "seed_big", dict(j, seeds={"bank": 2 ** 63 + 5, "mc": 7})
    yield "particles_float", dict(j, particles=64.0)
    yield "lambda_null", dict(j, **{"lambda": None})
    yield "eta_one", dict(j, eta=1.0)
    yield "rrt", dict(j, rrt={"trials": 10, "goal_bias": 0.1})
    yield "tracking", dict(j, tracking={"Q": 2.0, "R": [1, 2, 3][: len(j["workspace"]["bounds"]["lo"])]})
    ws = dict(j["workspace"])
    yield "obstacles_null", dict(j, workspace=dict(ws, obstacles=None))
    yield "obstacles_empty", dict(j, workspace=dict(ws, obstacles=[]))
    if ws.get("obstacles"):
        o = dict(ws["obstacles"][0])
        yield "box_extra", dict(j, workspace=dict(ws, obstacles=[dict(o, mid=1)] + ws["obstacles"][1:]))
        yield "box_inverted", dict(j, workspace=dict(ws, obstacles=[{"lo": o["hi"], "hi": o["lo"]}]))
        yield "box_short", dict(j, workspace=dict(ws, obstacles=[{"lo": o["lo"][:-1], "hi": o["hi"][:-1]}]))
    yield "start_in_goal_far", dict(j, start={"position": j["goal"]["lo"]})
    yield "goal_speed_neg", dict(j, goal=dict(j["goal"], max_speed=-1))


def test_fast_reader_equals_loader(checker, tmp_path):
    files = sorted(glob.glob(os.path.join(ROOT, "scenarios", "*.json")) +
                   glob.glob(os.path.join(ROOT, "tests", "golden", "scenarios", "*.json")))
    assert files
    paths = []
    for f in files:
        j = json.load(open(f))
        for tag, m in mutations(j):
            p = tmp_path / f"{os.path.basename(f)}.{tag}.json"
            p.write_text(json.dumps(m, indent=1 if tag == "pretty" else None))
            paths.append(str(p))
        raw = open(f).read()
        for tag, txt in (("dupkey", raw.replace("{", '{"dt": 0.3, ', 1)), ("trailing", raw + " x"),
                         ("comment", "// c\n" + raw), ("leading0", raw.replace('"samples": ', '"samples": 0', 1)),
                         ("bom", "﻿" + raw), ("crlf", raw.replace("\n", "\r\n"))):
            p = tmp_path / f"{os.path.basename(f)}.{tag}.json"
            p.write_text(txt)
            paths.append(str(p))
    r = subprocess.run([checker] + paths, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]
    lines = r.stdout.splitlines()
    accepted = [l for l in lines if l.startswith("accepted")]
    # every unmodified bundled scenario takes the fast path
    for f in files:
        assert any(l.endswith(f"{os.path.basename(f)}.same.json") for l in accepted), f
