import sys, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
n = 1000
iu = np.triu_indices(n, 1)
g = mb.DataGraph.from_edges(n, np.stack(iu, axis=1))
star9 = mb.QueryPlan(10, [(0, i) for i in range(1, 10)])
print(star9.canonical())
try:
    print(mb.count_colorful(g, star9, mb.random_coloring(g, 10, 1)))
except Exception as e:
    print(type(e), e)
