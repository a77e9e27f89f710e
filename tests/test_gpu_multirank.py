"""Multi-rank solves through the library on one B200 (the
analogue of the reference's 1-vs-8-workers record equality,
test_plan.cpp:188-227 and acceptance.cpp:435-471).

World 2 and 3 processes (torch.distributed gloo) each drive run_pump /
build_graph with the library's sharding on: graph rows [n r/W, n (r+1)/W)
built per rank and gathered, MC rollouts [n r/W, n (r+1)/W) certified per rank
with the int64 hit counts summed.  The collectives are the process group's
own, injected with pump_ctx_set_collectives (NCCL cannot put two ranks on one
GPU); every code path of the sharded solve but the NCCL transport runs.
Every rank's result must equal the single-process solve bit for bit."""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, scenario_text

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _text(name):
    j = json.loads(scenario_text(name))
    if name.startswith("quad3d"):
        j["samples"] = 700
    j["mc_samples"] = 3001  # not divisible by 2 or 3: uneven rollout shards
    return json.dumps(j)


KEYS = ("success", "partial_plans", "cost", "certified_cp", "smoothing_s", "n_edges", "n_plans")
ARRAYS = ("path", "pareto_cost", "pareto_cp", "mc_eval_ids", "mc_eval_values", "traj_pos", "traj_vel")


def _summary(r, g):
    out = {k: r[k] for k in KEYS}
    for k in ARRAYS:
        out[k] = np.ascontiguousarray(r[k]).tobytes()
    for k in ("row_ptr", "edge_to", "edge_cost", "hs_a", "hs_b", "edge_wp_off", "wp_hs_off"):
        out["g_" + k] = np.ascontiguousarray(g[k]).tobytes()
    return out


def _solve(name, api, ctx):
    txt = _text(name)
    sc = api.parse_scenario(txt)
    r = api.run_pump(sc, ctx=ctx)
    pos, vel = sc.nodes()
    p = sc.params()
    g = api.build_graph(pos, vel, sc.workspace(), sc.goal(), p["r_n"], p["dt"], p["eps_cc"], p["tau_max"],
                        ctx=ctx).export()
    return _summary(r, g)


def _worker(rank, world, port, names, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1607_06886_b200 import api

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = api.Context(0)
    api.set_collectives(ctx, rank, world)
    res = {n: _solve(n, api, ctx) for n in names}
    out.put((rank, res, ctx.io_counters()["collectives"]))
    dist.barrier()
    dist.destroy_process_group()


NAMES = ["three_obstacle", "quad3d_three_obstacle", "quad3d_indoor"]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_equals_single_rank(world):
    import sys

    sys.path.insert(0, ROOT)
    from paper_1607_06886_b200 import api

    ctx = api.Context(0)
    ref = {n: _solve(n, api, ctx) for n in NAMES}
    ctx.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, world, port, NAMES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, res, n_coll in got:
        assert n_coll >= 2 * len(NAMES), (rank, n_coll)  # the sharded paths really exchanged
        for n in NAMES:
            for k, v in ref[n].items():
                assert res[n][k] == v, (world, rank, n, k)
