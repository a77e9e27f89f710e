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


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["minimal", "three_obstacle"])
def test_cp_compare_matches_reference(tmp_path, name):
    """pump cp-compare (compare.hpp:38-96, pump_cli.cpp:77-90): the CSV rows
    against the reference's own cp_compare compiled in place (oracle/_ref).
    Analytical estimators (additive, multiplicative, conditional) to 1e-12;
    the MC and HSMC rows use portable normals here and glibc log/cos in the
    reference build, so they may differ by a flipped rollout or particle."""
    import ctypes as C

    import numpy as np

    ref_so = os.path.join(ROOT, "oracle", "_ref", "libpumpref.so")
    if not os.path.exists(ref_so):
        pytest.skip("reference not built (needs /root/reference)")
    sc = os.path.join(SCEN, name + ".json")
    r = run("plan", "--scenario", sc, "--out", str(tmp_path / "plan"))
    assert r.returncode == 0, r.stderr
    traj = tmp_path / "plan" / "trajectory.json"
    counts, n_mc = [8, 16, 40], 3000
    r = run("cp-compare", "--scenario", sc, "--trajectory", str(traj), "--waypoints", *map(str, counts),
            "--mc-samples", str(n_mc), "--out", str(tmp_path / "cmp"))
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "cmp" / "cp_compare.csv").read_text().splitlines()
    assert lines[0] == "method,waypoints,estimate,mc_reference,wall_time"
    rows = [ln.split(",") for ln in lines[1:]]
    methods = ["mc", "additive", "multiplicative", "conditional_multiplicative", "hsmc"]
    assert [x[0] for x in rows] == methods * len(counts)
    assert [int(x[1]) for x in rows] == [c for c in counts for _ in methods]
    L = C.CDLL(ref_so)
    L.ref_last_error.restype = C.c_char_p
    text = open(sc).read()
    particles = json.loads(text)["particles"]
    est = np.zeros(5 * len(counts))
    cnt = np.array(counts, dtype=np.int32)
    rc = L.ref_cp_compare(text.encode(), traj.read_text().encode(), cnt.ctypes.data_as(C.c_void_p), len(counts),
                          particles, n_mc, 4, est.ctypes.data_as(C.c_void_p))
    assert rc == 0, L.ref_last_error()
    for i, x in enumerate(rows):
        got, exp = float(x[2]), est[i]
        if x[0] == "mc":
            assert abs(got - exp) <= 2.0 / n_mc, (x, exp)
            assert float(x[3]) == got
        elif x[0] == "hsmc":
            assert abs(got - exp) <= 2.0 / particles, (x, exp)
        else:
            assert abs(got - exp) <= 1e-12 * max(1.0, abs(exp)), (x, exp)


def _ref_render(kind, scenario_path, report_path, traj_path):
    """The reference's own writers (oracle/_ref: report.hpp compiled in place)
    on the values read back from our files."""
    import ctypes as C

    lib = os.path.join(ROOT, "oracle", "_ref", "libpumpref.so")
    if not os.path.exists(lib):
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(lib)
    L.ref_render.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.c_long,
                             C.POINTER(C.c_long)]
    L.ref_last_error.restype = C.c_char_p
    args = [open(scenario_path).read().encode(), open(report_path).read().encode(),
            open(traj_path).read().encode() if traj_path and os.path.exists(traj_path) else b""]
    n = C.c_long()
    assert L.ref_render(kind, *args, 1, None, 0, C.byref(n)) == 0, L.ref_last_error()
    buf = C.create_string_buffer(n.value + 1)
    assert L.ref_render(kind, *args, 1, buf, n.value + 1, C.byref(n)) == 0
    return buf.raw[:n.value].split(b"\x1f")


@pytest.mark.gpu
@pytest.mark.parametrize("scenario", ["minimal.json", "three_obstacle.json"])
def test_writers_byte_equal_to_reference_writers(tmp_path, scenario):
    """report.json / pareto.csv / trajectory.json (plan), report.json +
    trajectory.json (rrt) and report.json (certify) equal, byte for byte, what
    the reference's own writers (report.hpp:31-129, pump_cli.cpp:48-109) emit
    for the same result values -- timings included."""
    sc = os.path.join(SCEN, scenario)
    out = tmp_path / "plan"
    r = run("plan", "--scenario", sc, "--out", str(out))
    assert r.returncode in (0, 2), r.stderr
    ref = _ref_render(0, sc, out / "report.json", out / "trajectory.json")
    assert ref[0] == (out / "report.json").read_bytes()
    assert ref[1] == (out / "pareto.csv").read_bytes()
    if (out / "trajectory.json").exists():
        assert ref[2] == (out / "trajectory.json").read_bytes()
        c = run("certify", "--scenario", sc, "--trajectory", str(out / "trajectory.json"), "--out",
                str(tmp_path / "cert"))
        assert c.returncode in (0, 2), c.stderr
        assert _ref_render(2, sc, tmp_path / "cert" / "report.json", None)[0] == \
            (tmp_path / "cert" / "report.json").read_bytes()
    rr = run("rrt", "--scenario", sc, "--out", str(tmp_path / "rrt"))
    assert rr.returncode in (0, 2), rr.stderr
    ref = _ref_render(1, sc, tmp_path / "rrt" / "report.json", tmp_path / "rrt" / "trajectory.json")
    assert ref[0] == (tmp_path / "rrt" / "report.json").read_bytes()
    if (tmp_path / "rrt" / "trajectory.json").exists():
        assert ref[1] == (tmp_path / "rrt" / "trajectory.json").read_bytes()
