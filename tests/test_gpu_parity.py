"""GPU parity: colourful counts from the CUDA engine (through the C ABI) are
bit-identical to the CPU oracle (brute force) and the compiled reference
engine on the same graph, query and colouring seed."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TRIANGLE_FAMILY = {
    "edge": (2, [(0, 1)]),
    "p3": (3, [(0, 1), (1, 2)]),
    "p4": (4, [(0, 1), (1, 2), (2, 3)]),
    "star4": (5, [(0, 1), (0, 2), (0, 3), (0, 4)]),
    "c3": (3, [(0, 1), (1, 2), (2, 0)]),
    "tri_pendant": (4, [(0, 1), (1, 2), (2, 3), (3, 1)]),
    "q6": (6, [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2), (2, 4), (4, 5)]),
    "diamond": (4, [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2)]),
    "bowtie": (5, [(0, 1), (1, 2), (2, 0), (0, 3), (3, 4), (4, 0)]),
    "book3": (5, [(0, 1), (0, 2), (1, 2), (0, 3), (1, 3), (0, 4), (1, 4)]),
}


def _ref_count(reference, g, k, qedges, chi, tree=-1):
    rg = reference.graph(g.num_vertices(), g.edges())
    return reference.count(rg, reference.plan(k, qedges), chi, engine=1, tree=tree)


@pytest.mark.parametrize("name", sorted(TRIANGLE_FAMILY))
def test_small_against_brute_force(mb, oracle, name):
    k, q = TRIANGLE_FAMILY[name]
    plan = mb.QueryPlan(k, q)
    for gseed in range(3):
        g = mb.DataGraph.erdos_renyi(14, 40, seed=gseed)
        off, adj = g.csr()
        for cseed in range(3):
            chi = mb.random_coloring(g, k, 31 * gseed + cseed)
            assert mb.count_colorful(g, plan, chi) == oracle.brute(off, adj, k, q, chi)


@pytest.mark.parametrize("name", sorted(TRIANGLE_FAMILY))
def test_against_reference_engine(mb, reference, name):
    k, q = TRIANGLE_FAMILY[name]
    plan = mb.QueryPlan(k, q)
    g = mb.DataGraph.chung_lu(3000, 2.1, 10.0, seed=11)
    chi = np.stack([mb.random_coloring(g, k, s) for s in (100, 101, 102)])
    got = mb.count_colorful(g, plan, chi)
    for i, s in enumerate((100, 101, 102)):
        assert int(got[i]) == _ref_count(reference, g, k, q, chi[i])


def test_every_tree_same_count(mb, reference):
    k, q = TRIANGLE_FAMILY["q6"]
    plan = mb.QueryPlan(k, q)
    g = mb.DataGraph.chung_lu(2000, 2.1, 12.0, seed=5)
    chi = mb.random_coloring(g, k, 7)
    want = _ref_count(reference, g, k, q, chi)
    for t in range(plan.num_trees()):
        plan.use_tree(t)
        assert mb.count_colorful(g, plan, chi) == want, plan.canonical(t)


CYCLE_FAMILY = {
    "c4": (4, [(0, 1), (1, 2), (2, 3), (3, 0)]),
    "c5": (5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)]),
    "c6": (6, [(i, (i + 1) % 6) for i in range(6)]),
    "c7": (7, [(i, (i + 1) % 7) for i in range(7)]),
    "c5_pendant": (6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (2, 5)]),
    "theta": (8, [(0, 1), (1, 2), (2, 7), (0, 3), (3, 4), (4, 7), (0, 5), (5, 6), (6, 7)]),
    # BASELINE config 4: 6-cycle with chords 0-2 and 3-5, path 1-6-7-8 and triangle 8-9-1 (14 edges)
    "sp10": (10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 2), (3, 5), (1, 6), (6, 7), (7, 8),
                  (8, 9), (9, 1), (1, 8)]),
    # the same without the chord 1-8 (a 5-cycle 1-6-7-8-9 instead of the triangle)
    "sp10_open": (10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 2), (3, 5), (1, 6), (6, 7), (7, 8),
                       (8, 9), (9, 1)]),
    "brain1": (9, [(0, 1), (1, 2), (2, 3), (3, 0), (0, 4), (4, 5), (5, 6), (6, 7), (7, 8), (8, 0)]),
    "sat": (11, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (0, 5), (2, 6), (5, 6), (5, 7), (5, 8), (6, 8),
                 (8, 9), (9, 10), (10, 8)]),
    "k4_minus": (4, [(0, 1), (1, 2), (2, 3), (3, 0), (0, 2)]),
}


@pytest.mark.parametrize("name", sorted(CYCLE_FAMILY))
def test_cycles_against_brute_force(mb, oracle, name):
    k, q = CYCLE_FAMILY[name]
    plan = mb.QueryPlan(k, q)
    n = 12 if k <= 8 else 14
    for gseed in range(2):
        g = mb.DataGraph.erdos_renyi(n, 3 * n, seed=100 + gseed)
        off, adj = g.csr()
        for cseed in range(2):
            chi = mb.random_coloring(g, k, 7 * gseed + cseed)
            assert mb.count_colorful(g, plan, chi) == oracle.brute(off, adj, k, q, chi), (gseed, cseed)


@pytest.mark.parametrize("name", sorted(CYCLE_FAMILY))
def test_cycles_against_reference_engine(mb, reference, name):
    k, q = CYCLE_FAMILY[name]
    plan = mb.QueryPlan(k, q)
    g = mb.DataGraph.chung_lu(400 if k >= 8 else 1500, 2.1, 8.0, seed=21)
    for s in (100, 101):
        chi = mb.random_coloring(g, k, s)
        assert mb.count_colorful(g, plan, chi) == _ref_count(reference, g, k, q, chi)


@pytest.mark.parametrize("name", ["sat", "sp10", "theta", "brain1"])
def test_cycle_plans_every_tree(mb, reference, name):
    k, q = CYCLE_FAMILY[name]
    plan = mb.QueryPlan(k, q)
    g = mb.DataGraph.chung_lu(300, 2.1, 7.0, seed=3)
    chi = mb.random_coloring(g, k, 9)
    want = _ref_count(reference, g, k, q, chi)
    for t in range(plan.num_trees()):
        plan.use_tree(t)
        assert mb.count_colorful(g, plan, chi) == want, plan.canonical(t)


def test_device_colourings_are_the_reference_colourings(mb):
    """count_colorful_seeds / estimate generate their colourings on the device
    (k_random_colorings: one warp per mt19937_64 stream).  They must be the
    reference's random_coloring byte for byte (graph.cpp:142-151), for sizes
    around the generator's 312-word state and every k, and also when draws are
    rejected: with the rejection limit forced to 2^63 about half of the draws
    are skipped, and the expected colours follow from the raw stream of the
    oracle's generator (pinned to std::mt19937_64 in tests/test_oracle.py)."""
    from oracle import Oracle

    O = Oracle()
    for n in (1, 311, 312, 313, 1000, 100003):
        g = mb.DataGraph.from_edges(n, np.zeros((0, 2), dtype=np.int64))
        for k in (1, 2, 3, 6, 7, 10, 16, 32):
            seeds = [7, 100, 2**63 + 5, 0]
            got = mb.device_random_colorings(g, k, seeds)
            for i, s in enumerate(seeds):
                assert np.array_equal(got[i], mb.random_coloring(g, k, s)), (n, k, s)
        limit = 1 << 63
        seeds = [3, 4]
        got = mb.device_random_colorings(g, 6, seeds, limit=limit)
        for i, s in enumerate(seeds):
            raw = O.mt64(s, 4 * n + 64)
            acc = raw[raw < np.uint64(limit)][:n]
            assert len(acc) == n
            assert np.array_equal(got[i], (1 + acc % np.uint64(6)).astype(np.uint8)), (n, s)


def test_seeded_counts_equal_counts_of_host_colourings(mb):
    g = mb.DataGraph.chung_lu(3000, 2.1, 8.0, 11)
    seeds = list(range(40, 53))  # 13: one full batch of 8 and a partial one
    for k, q in ((6, [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2), (2, 4), (4, 5)]), (5, [(i, (i + 1) % 5) for i in range(5)])):
        plan = mb.QueryPlan(k, q)
        chis = np.stack([mb.random_coloring(g, k, s) for s in seeds])
        assert np.array_equal(mb.count_colorful_seeds(g, plan, seeds), mb.count_colorful(g, plan, chis))
