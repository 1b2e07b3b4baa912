"""Two processes driving the REAL engine (both ranks on cuda:0, gloo for the
plumbing; the driver's boxes have one GPU): the vertex-sharded count and the
colouring-sharded estimate must equal the single-process results."""
import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


QUERIES = {
    "c5": (5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)]),
    "c7": (7, [(i, (i + 1) % 7) for i in range(7)]),
    "c5_pendant": (6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (2, 5)]),
    "q6": (6, [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2), (2, 4), (4, 5)]),
    # the pair-producing 6-cycle block is sharded, every rank streams its
    # partial pair table through the whole root
    "theta": (8, [(0, 1), (1, 2), (2, 7), (0, 3), (3, 4), (4, 7), (0, 5), (5, 6), (6, 7)]),
}


def _worker(rank, world, port, results):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1602_04478_b200 as mb
        from paper_1602_04478_b200 import parallel

        g = mb.DataGraph.chung_lu(3000, 2.1, 8.0, 11)
        out = {}
        for name, (k, q) in QUERIES.items():
            plan = mb.QueryPlan(k, q)
            chis = np.stack([mb.random_coloring(g, k, s) for s in (3, 4, 5)])
            part, split = mb.count_colorful_shard(g, plan, chis, rank, world)
            tot = parallel.distributed_count_vertex_sharded(g, plan, chis, device="cpu")
            out[name] = ([int(x) for x in part], split, [int(x) for x in tot], mb.engine_device(g))
        plan = mb.QueryPlan(*QUERIES["c5"])
        rep = parallel.distributed_estimate(g, plan, mb.DB, 9, 77, device="cpu")
        out["estimate"] = (rep.per_trial_colorful, rep.mean_estimate, rep.cv)
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_two_processes_real_engine(mb):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    g = mb.DataGraph.chung_lu(3000, 2.1, 8.0, 11)
    for name, (k, q) in QUERIES.items():
        plan = mb.QueryPlan(k, q)
        chis = np.stack([mb.random_coloring(g, k, s) for s in (3, 4, 5)])
        want = [int(x) for x in mb.count_colorful(g, plan, chis)]
        p0, s0, t0, d0 = results[0][name]
        p1, s1, t1, d1 = results[1][name]
        assert t0 == want and t1 == want, name
        assert [a + b for a, b in zip(p0, p1)] == want, name
        assert d0 == 0 and d1 == 0
        if name in ("c5", "c7", "theta"):  # root cycle blocks with a scalar output are split
            assert s0 and s1 and all(a > 0 for a in p0) and all(b > 0 for b in p1), name
    rep = mb.estimate(g, mb.QueryPlan(*QUERIES["c5"]), mb.DB, 9, 77)
    for r in (0, 1):
        per, mean, cv = results[r]["estimate"]
        assert per == rep.per_trial_colorful and mean == rep.mean_estimate and cv == rep.cv
