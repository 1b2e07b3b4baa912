import sys
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
from oracle import Oracle
O = Oracle()
cases = {
 'diamond': (4, [(0,1),(1,2),(2,0),(1,3),(3,2)]),
 'book3': (5, [(0,1),(0,2),(1,2),(0,3),(1,3),(0,4),(1,4)]),
 'diamond_tail': (5, [(0,1),(1,2),(2,0),(1,3),(3,2),(0,4)]),
 'q6': (6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)]),
}
g = mb.DataGraph.erdos_renyi(14, 40, seed=0)
off, adj = g.csr()
for name, (k, q) in cases.items():
    p = mb.QueryPlan(k, q)
    chi = mb.random_coloring(g, k, 0)
    try:
        print(name, p.canonical(), mb.count_colorful(g, p, chi), O.brute(off, adj, k, q, chi), flush=True)
    except Exception as e:
        print(name, p.canonical(), "ERR", e, flush=True)
        break
