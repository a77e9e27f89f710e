"""Multi-process (gloo, world_size 2/3) check of the sharded MC certification
on CPU: every rank simulates its rollout range [n r/W, n (r+1)/W) (the
library's partition, pump_shard_range) and an integer all-reduce of the hit
counts must reproduce the single-process count exactly."""
import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, scenario_text


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _traj_and_models():
    import oracle

    txt = scenario_text("quad3d_three_obstacle")
    cl, sc = oracle.scenario_models(txt)
    j = json.loads(txt)
    ws = {"bounds_lo": j["workspace"]["bounds"]["lo"], "bounds_hi": j["workspace"]["bounds"]["hi"],
          "obs_lo": [o["lo"] for o in j["workspace"]["obstacles"]],
          "obs_hi": [o["hi"] for o in j["workspace"]["obstacles"]]}
    y = np.linspace([1.0, 5.0, 2.0], [2.47, 6.0, 2.0], 60)
    return cl, ws, y, sc["eps_cc"]


def _worker(rank, world, port, n_mc, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch

    import oracle
    from paper_1607_06886_b200 import api

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cl, ws, y, eps = _traj_and_models()
    lo, hi = api.shard_range(n_mc, rank, world)
    hits = oracle.mc_hits(cl, ws, y, lo, hi, 2, eps, workers=1)
    t = torch.tensor([hits], dtype=torch.int64)
    dist.all_reduce(t)
    sizes = torch.tensor([hi - lo], dtype=torch.int64)
    dist.all_reduce(sizes)
    if rank == 0:
        out.put((int(t.item()), int(sizes.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_mc_equals_single_process(oracle_lib, world):
    n_mc = 3001
    cl, ws, y, eps = _traj_and_models()
    full = oracle_lib.mc_hits(cl, ws, y, 0, n_mc, 2, eps, workers=4)
    assert 0 < full < n_mc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_mc, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    total, covered = q.get(timeout=10)
    assert covered == n_mc
    assert total == full


def test_shard_range_partition_matches_library():
    from paper_1607_06886_b200 import api
    import ctypes as C

    L = api.lib()
    for n in (0, 1, 7, 20000, 10 ** 7 + 3):
        for world in (1, 2, 3, 8):
            spans = []
            for r in range(world):
                lo, hi = C.c_int64(), C.c_int64()
                assert L.pump_shard_range(n, r, world, C.byref(lo), C.byref(hi)) == 0
                assert (lo.value, hi.value) == api.shard_range(n, r, world)
                spans.append((lo.value, hi.value))
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
