"""The pump CLI (tools/pump, drop-in for tools/pump_cli.cpp) and the C++
drop-in API driver (tests/cpp/test_dropin.cpp).  Ports tests/cli_smoke.sh:
exit codes, emitted files, byte-stable outputs, certify round trip."""
import json
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

PUMP = os.path.join(ROOT, "tools", "pump")
DROPIN = os.path.join(ROOT, "tools", "test_dropin")
SCEN = os.path.join(GOLDEN, "scenarios")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not (os.path.exists(PUMP) and os.path.exists(DROPIN)):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)


def run(*args, cwd=None):
    return subprocess.run([PUMP, *args], capture_output=True, text=True, cwd=cwd, timeout=600)


def test_input_errors_exit_1(tmp_path):
    """cli_smoke.sh:11-19 (no GPU needed: the scenario fails to load first)."""
    r = run("plan", "--scenario", str(tmp_path / "nope.json"), "--out", str(tmp_path / "a"))
    assert r.returncode == 1
    bad = tmp_path / "bad.json"
    bad.write_text('{"alpha": 2}')
    r = run("plan", "--scenario", str(bad), "--out", str(tmp_path / "a"))
    assert r.returncode == 1 and "missing required key" in r.stderr
    assert run("plan").returncode == 1
    assert run("frobnicate", "--scenario", str(bad)).returncode == 1


@pytest.mark.gpu
def test_plan_outputs_stable_and_certify_round_trip(tmp_path):
    """cli_smoke.sh:21-58."""
    sc = os.path.join(SCEN, "minimal.json")
    r = run("plan", "--scenario", sc, "--out", str(tmp_path / "plan"))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("success cost=")
    for f in ("report.json", "pareto.csv", "trajectory.json"):
        assert (tmp_path / "plan" / f).stat().st_size > 0
    r2 = run("plan", "--scenario", sc, "--out", str(tmp_path / "plan2"))
    assert r2.returncode == 0

    def strip(p):
        return [ln for ln in p.read_text().splitlines() if "_seconds" not in ln]

    assert strip(tmp_path / "plan" / "report.json") == strip(tmp_path / "plan2" / "report.json")
    for f in ("pareto.csv", "trajectory.json"):
        assert (tmp_path / "plan" / f).read_bytes() == (tmp_path / "plan2" / f).read_bytes()
    assert (tmp_path / "plan" / "pareto.csv").read_text().splitlines()[0] == "cost,cp_hat"
    c = run("certify", "--scenario", sc, "--trajectory", str(tmp_path / "plan" / "trajectory.json"), "--out",
            str(tmp_path / "cert"))
    assert c.returncode == 0, c.stderr
    planned = json.loads((tmp_path / "plan" / "report.json").read_text())["certified_cp"]
    certified = json.loads((tmp_path / "cert" / "report.json").read_text())["certified_cp"]
    assert planned == certified
    c2 = run("certify", "--scenario", sc, "--trajectory", str(tmp_path / "plan" / "trajectory.json"), "--out",
             str(tmp_path / "cert2"))
    assert (tmp_path / "cert" / "report.json").read_bytes() == (tmp_path / "cert2" / "report.json").read_bytes()


@pytest.mark.gpu
def test_plan_matches_oracle(oracle_lib, tmp_path):
    sc = os.path.join(SCEN, "three_obstacle.json")
    r = run("plan", "--scenario", sc, "--out", str(tmp_path / "p"))
    assert r.returncode == 0, r.stderr
    rep = json.loads((tmp_path / "p" / "report.json").read_text())
    with open(sc) as f:
        o = oracle_lib.run_pump(f.read(), workers=os.cpu_count() or 4)
    assert rep["path"] == o["path"].tolist()
    assert rep["certified_cp"] == o["certified_cp"] and rep["cost"] == o["cost"]
    assert rep["partial_plans"] == o["partial_plans"]
    assert [e["plan"] for e in rep["mc_evaluations"]] == o["mc_eval_ids"].tolist()


@pytest.mark.gpu
def test_cpp_dropin_api():
    r = subprocess.run([DROPIN, SCEN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_rrt_subcommand_matches_oracle(oracle_lib, tmp_path):
    """pump rrt (pump_cli.cpp:63-76): report fields equal the oracle's
    repeated_rrt with the scenario's trials / alpha / mc_samples."""
    sc = os.path.join(SCEN, "minimal.json")
    r = run("rrt", "--scenario", sc, "--out", str(tmp_path / "rrt"))
    assert r.returncode in (0, 2), r.stderr
    rep = json.loads((tmp_path / "rrt" / "report.json").read_text())
    assert rep["algorithm"] == "rrt"
    with open(sc) as f:
        o = oracle_lib.repeated_rrt(f.read(), workers=os.cpu_count() or 4)
    assert rep["success"] == o["success"] and (r.returncode == 0) == o["success"]
    assert rep["trials_reaching_goal"] == o["trials_reaching_goal"]
    assert rep["certification_attempts"] == o["certification_attempts"]
    assert rep["cost"] == o["cost"] and rep["certified_cp"] == o["certified_cp"]
    assert (tmp_path / "rrt" / "trajectory.json").exists() == o["success"]
