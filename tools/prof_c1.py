# short config-1 run for ncu: 1 warm-up count + 1 profiled count of 2 colourings
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
g = mb.DataGraph.chung_lu(1000000, 2.1, 16.0, seed=2)
plan = mb.QueryPlan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chi = np.stack([mb.random_coloring(g, 6, s) for s in range(100, 108)])
print(mb.count_colorful(g, plan, chi))
