"""The library's host-side geometry / steering helpers (the same
__host__ __device__ code the kernels run) against the CPU oracle, bit for
bit, on random worlds.  CPU only: these entry points need no GPU.

Covers the exact-preserving rewrites inside that shared code: the single
min-corner prune test of local_convex_region (geom.hpp:189-225), the span
pruning and obstacle culling of motion_collides (geom.hpp:96-123), and the
connect() scan + golden section (steer.hpp:111-182)."""
import numpy as np
import pytest

from paper_1607_06886_b200 import api


def _world(rng, dw, n_obs):
    lo = np.zeros(dw)
    hi = np.full(dw, 10.0)
    c = rng.uniform(1.0, 9.0, size=(n_obs, dw))
    h = rng.uniform(0.2, 1.5, size=(n_obs, dw))
    return {"bounds_lo": lo, "bounds_hi": hi, "obs_lo": c - h, "obs_hi": c + h}


@pytest.mark.parametrize("dw", [2, 3])
def test_local_convex_region_matches_oracle(oracle_lib, dw):
    rng = np.random.default_rng(11 + dw)
    checked = 0
    for trial in range(60):
        ws = _world(rng, dw, int(rng.integers(1, 24)))
        for _ in range(20):
            y = rng.uniform(0.0, 10.0, size=dw)
            if not oracle_lib.point_free(ws, y):
                continue
            yd = rng.normal(size=dw) * (0.0 if trial % 7 == 0 else 1.0)
            try:
                ea, eb, ef = oracle_lib.local_convex_region(ws, y, yd)
            except Exception as e:  # the reference's runtime_error: the library must raise too
                with pytest.raises(api.PumpError):
                    api.local_convex_region(ws, y, yd)
                continue
            ga, gb, gf = api.local_convex_region(ws, y, yd)
            assert ga.view(np.uint64).tolist() == ea.view(np.uint64).tolist()
            assert gb.view(np.uint64).tolist() == eb.view(np.uint64).tolist()
            assert gf.tolist() == ef.tolist()
            checked += 1
    assert checked > 300


@pytest.mark.parametrize("dw", [2, 3])
def test_connect_and_motion_collides_match_oracle(oracle_lib, dw):
    rng = np.random.default_rng(5 + dw)
    ws = _world(rng, dw, 12)
    n_hit = n_free = 0
    for trial in range(1500):
        ap, bp = rng.uniform(0.5, 9.5, size=(2, dw))
        av, bv = rng.normal(size=(2, dw))
        if trial % 5 == 1:  # near-equal states / aligned motion: flat cost curves, near-ties
            bp = ap + rng.normal(size=dw) * 1e-3
            bv = av + rng.normal(size=dw) * 1e-4
        elif trial % 5 == 2:
            av = np.zeros(dw)
            bv = np.zeros(dw)
        elif trial % 5 == 3:
            bp = ap + av * rng.uniform(0.1, 3.0)
        g = api.connect(ap, av, bp, bv, 5.0)
        e = oracle_lib.connect(ap, av, bp, bv, 5.0)
        assert g["ok"] == e["ok"]
        assert np.float64(g["tau"]).tobytes() == np.float64(e["tau"]).tobytes()
        assert np.float64(g["cost"]).tobytes() == np.float64(e["cost"]).tobytes()
        assert api.steer_cost(ap, av, bp, bv, 0.7) == oracle_lib.steer_cost(ap, av, bp, bv, 0.7)
        if not e["ok"]:
            continue
        for eps in (0.05, 0.5):
            got = api.motion_collides(ws, ap, av, bp, bv, e["tau"], e["acc0"], e["jerk"], eps)
            exp = oracle_lib.motion_collides(ws, ap, av, bp, bv, e["tau"], e["acc0"], e["jerk"], eps)
            assert got == exp
            n_hit += exp
            n_free += not exp
    assert n_hit > 20 and n_free > 20


def test_connect_lazy_decisions_stress(oracle_lib):
    """connect()'s lazily decided comparisons (cubic in 1/tau within kLazyErr S,
    steer_cost only when ambiguous) against the literal scan + golden section
    on 20000 pairs across scales: flat cost curves, near-ties, cancellation."""
    rng = np.random.default_rng(11)
    for trial in range(20000):
        dw = 2 + trial % 2
        scale = 10.0 ** rng.uniform(-3, 3)
        ap = rng.uniform(-1, 1, size=dw) * scale
        av = rng.normal(size=dw) * 10.0 ** rng.uniform(-3, 1)
        kind = trial % 6
        if kind == 0:
            bp, bv = ap + rng.normal(size=dw) * scale, rng.normal(size=dw)
        elif kind == 1:  # nearly identical states
            bp, bv = ap + rng.normal(size=dw) * scale * 1e-7, av + rng.normal(size=dw) * 1e-7
        elif kind == 2:  # the straight line the start velocity follows
            bp, bv = ap + av * rng.uniform(0.01, 10.0), av.copy()
        elif kind == 3:  # offsets far below the positions' magnitude (cancellation in dp)
            bp = ap + rng.normal(size=dw) * 1e-9 * scale
            bv = rng.normal(size=dw) * 1e-3
        elif kind == 4:
            bp, bv = ap + rng.normal(size=dw) * scale, np.zeros(dw)
            av = np.zeros(dw)
        else:
            bp, bv = ap + rng.normal(size=dw), -av
        tau_max = 10.0 ** rng.uniform(-1, 2)
        g = api.connect(ap, av, bp, bv, tau_max)
        e = oracle_lib.connect(ap, av, bp, bv, tau_max)
        assert g["ok"] == e["ok"], trial
        assert np.float64(g["tau"]).tobytes() == np.float64(e["tau"]).tobytes(), trial
        assert np.float64(g["cost"]).tobytes() == np.float64(e["cost"]).tobytes(), trial


@pytest.mark.parametrize("name", ["minimal", "three_obstacle", "quad3d_three_obstacle"])
def test_scenario_nodes_match_oracle(oracle_lib, name):
    """The node set run_pump plans over (pump.hpp:184-189, sample.hpp:56-89)."""
    from conftest import scenario_text

    txt = scenario_text(name)
    pos, vel = api.parse_scenario(txt).nodes()
    epos, evel = oracle_lib.scenario_nodes(txt)
    assert pos.view(np.uint64).tolist() == np.asarray(epos).view(np.uint64).tolist()
    assert vel.view(np.uint64).tolist() == np.asarray(evel).view(np.uint64).tolist()
