import sys
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
from oracle import Oracle
O = Oracle()
q = [(0,1),(0,2),(1,2),(0,3),(1,3),(0,4),(1,4)]
p = mb.QueryPlan(5, q)
g = mb.DataGraph.erdos_renyi(14, 40, seed=0)
off, adj = g.csr()
chi = mb.random_coloring(g, 5, 0)
try:
    print(mb.count_colorful(g, p, chi), O.brute(off, adj, 5, q, chi))
except Exception as e:
    print("ERR", e)
