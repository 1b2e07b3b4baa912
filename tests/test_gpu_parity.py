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
