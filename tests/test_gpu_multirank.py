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
    # leaf blocks only: with the table exchange every level is sharded and the
    # root leaf's rows are totalled per rank
    "path5": (5, [(0, 1), (1, 2), (2, 3), (3, 4)]),
    "star_path": (6, [(0, 1), (0, 2), (0, 3), (3, 4), (4, 5)]),
    # triangle with pendant trees: leaf tables feed a 3-cycle root
    "tri_tails": (6, [(0, 1), (1, 2), (2, 0), (0, 3), (1, 4), (4, 5)]),
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
            # the same with the leaf blocks sharded and their rows exchanged
            # (gloo: staged through the host; both ranks share cuda:0)
            ag = parallel.make_allgather(dist, world, rank)
            xpart, xsplit = mb.count_colorful_sharded(g, plan, chis, rank, world, ag)
            xtot = parallel.distributed_count_vertex_sharded(g, plan, chis, device="cpu", exchange=True)
            out[name] = ([int(x) for x in part], split, [int(x) for x in tot], mb.engine_device(g),
                         [int(x) for x in xpart], xsplit, [int(x) for x in xtot])
            out[name + "/bytes"] = mb.engine_exchanged_bytes(g)
        plan = mb.QueryPlan(*QUERIES["c5"])
        rep = parallel.distributed_estimate(g, plan, mb.DB, 9, 77, device="cpu")
        out["estimate"] = (rep.per_trial_colorful, rep.mean_estimate, rep.cv)
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_processes_real_engine(mb, world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    g = mb.DataGraph.chung_lu(3000, 2.1, 8.0, 11)
    for name, (k, q) in QUERIES.items():
        plan = mb.QueryPlan(k, q)
        chis = np.stack([mb.random_coloring(g, k, s) for s in (3, 4, 5)])
        want = [int(x) for x in mb.count_colorful(g, plan, chis)]
        rows = [results[r][name] for r in range(world)]
        parts, splits = [r[0] for r in rows], [r[1] for r in rows]
        assert all(r[2] == want for r in rows), name
        assert [sum(col) for col in zip(*parts)] == want, name
        assert all(r[3] == 0 for r in rows)
        # root cycle blocks with a scalar output are split by anchor, root
        # 3-cycle blocks on the relative-colour kernel by warp batch
        if name in ("c5", "c7", "theta", "q6"):
            assert all(splits) and all(x > 0 for p in parts for x in p), name
        # with the table exchange: same totals, and leaf roots are split too
        xparts, xsplits = [r[4] for r in rows], [r[5] for r in rows]
        assert all(r[6] == want for r in rows), name
        assert [sum(col) for col in zip(*xparts)] == want, name
        assert len(set(xsplits)) == 1, name
        if name in ("c5", "c7", "theta", "q6", "path5", "star_path"):
            assert xsplits[0] and all(x > 0 for p in xparts for x in p), name
    # plans with leaf blocks below the root moved rows between the ranks
    for r in range(world):
        seen = 0
        for name in QUERIES:
            now = results[r][name + "/bytes"]
            if name in ("c5_pendant", "q6", "path5", "star_path", "tri_tails"):
                assert now > seen, name
            seen = now
    rep = mb.estimate(g, mb.QueryPlan(*QUERIES["c5"]), mb.DB, 9, 77)
    for r in range(world):
        per, mean, cv = results[r]["estimate"]
        assert per == rep.per_trial_colorful and mean == rep.mean_estimate and cv == rep.cv
