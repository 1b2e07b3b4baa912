"""Multi-rank plumbing (paper_1602_04478_b200.parallel) on CPU: world size 2
over gloo, with the oracle's brute-force count standing in for the device
call.  The gathered per-trial counts and the estimate report must equal the
reference's single-process estimate (tests/golden/estimates.json)."""
import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1602_04478_b200 as mb
        from paper_1602_04478_b200 import parallel
        from oracle import Oracle

        O = Oracle()
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "counts.json")))
        plans = json.load(open(os.path.join(ROOT, "tests", "golden", "plans.json")))
        est = json.load(open(os.path.join(ROOT, "tests", "golden", "estimates.json")))
        out = []
        for e in est:
            g = gold["graphs"][e["graph"]]
            p = plans[e["query"]]
            off, adj, _ = O.build_csr(g["n"], g["edges"])
            fn = lambda s, g=g, p=p, off=off, adj=adj: O.brute(off, adj, p["k"], p["edges"],
                                                               O.random_coloring(g["n"], p["k"], s))
            plan = mb.QueryPlan(p["k"], p["edges"])
            rep = parallel.distributed_estimate(None, plan, 1, e["trials"], e["seed"], count_fn=fn, device="cpu")
            out.append((rep.per_trial_colorful, rep.mean_estimate, rep.cv, rep.subgraph_estimate))
        # uneven shards: 3 seeds over 2 ranks, 1 seed over 2 ranks
        g = gold["graphs"]["er24"]
        off, adj, _ = O.build_csr(g["n"], g["edges"])
        c3 = [(0, 1), (1, 2), (2, 0)]
        fn = lambda s: O.brute(off, adj, 3, c3, O.random_coloring(g["n"], 3, s))
        three = parallel.distributed_count_seeds(None, None, [5, 6, 7], count_fn=fn, device="cpu")
        one = parallel.distributed_count_seeds(None, None, [9], count_fn=fn, device="cpu")
        results[rank] = (out, three.tolist(), one.tolist(), [fn(5), fn(6), fn(7)], [fn(9)])
    finally:
        dist.destroy_process_group()


def test_block_partition():
    from paper_1602_04478_b200.parallel import block

    for n in (0, 1, 7, 64, 1001):
        for w in (1, 2, 3, 8):
            spans = [block(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_two_ranks_gloo_estimate_matches_reference():
    est = json.load(open(os.path.join(ROOT, "tests", "golden", "estimates.json")))
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    for rank in (0, 1):
        out, three, one, three_want, one_want = results[rank]
        assert three == three_want and one == one_want
        for (per, mean, cv, sub), e in zip(out, est):
            assert per == e["per_trial"]
            # the mean is taken in long double through the C ABI, as the
            # reference's estimate() does: bit-identical doubles
            assert mean == e["mean"]
            assert cv == e["cv"]
            assert sub == e["subgraph"]


def _shard_worker(rank, world, port, results):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1602_04478_b200 import CountOverflowError, parallel
        from oracle import Oracle

        O = Oracle()
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "counts.json")))
        g = gold["graphs"]["skew60"]
        off, adj, _ = O.build_csr(g["n"], g["edges"])
        c5 = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)]
        chis = [O.random_coloring(g["n"], 5, s) for s in (1, 2)]
        want = [O.brute(off, adj, 5, c5, c) for c in chis]

        # each rank reports an uneven share of every colouring's count
        def fn(r, w):
            return [(x // 3 if r == 0 else x - x // 3) for x in want], False

        got = parallel.distributed_count_vertex_sharded(None, None, np.stack(chis), count_fn=fn, device="cpu")
        # partials whose sum passes 2^64 are the reference's OverflowError on every rank
        big = lambda r, w: ([(1 << 63) + 5], False)
        try:
            parallel.distributed_count_vertex_sharded(None, None, np.stack(chis[:1]), count_fn=big, device="cpu")
            over = "none"
        except CountOverflowError:
            over = "sum"
        # one rank overflowing alone is an overflow everywhere
        one = lambda r, w: ([0], r == 1)
        try:
            parallel.distributed_count_vertex_sharded(None, None, np.stack(chis[:1]), count_fn=one, device="cpu")
            over1 = "none"
        except CountOverflowError:
            over1 = "rank"
        # the table-exchange callback (parallel.make_allgather) on host memory:
        # this rank's packed rows sit in slice `rank`; afterwards every slice
        # holds its rank's rows
        nbytes = 4096 + 16
        xbuf = np.zeros(world * nbytes, np.uint8)
        xbuf[rank * nbytes:(rank + 1) * nbytes] = (np.arange(nbytes) * (rank + 3) + rank) % 251
        parallel.make_allgather(dist, world, rank, device="cpu")(xbuf.ctypes.data, nbytes, 0)
        xok = all(np.array_equal(xbuf[q * nbytes:(q + 1) * nbytes], (np.arange(nbytes) * (q + 3) + q) % 251)
                  for q in range(world))
        results[rank] = ([int(x) for x in got], want, over, over1, xok)
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo_vertex_sharded_sum():
    """Vertex-sharded counting plumbing (parallel.distributed_count_vertex_sharded):
    the ranks' partial counts are all-gathered and added with checked u64
    arithmetic; overflow on any rank or in the sum raises on every rank."""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_shard_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    for rank in (0, 1):
        got, want, over, over1, xok = results[rank]
        assert got == want
        assert over == "sum" and over1 == "rank"
        assert xok
