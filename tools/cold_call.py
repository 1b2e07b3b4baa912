import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
t=time.time(); g = mb.DataGraph.chung_lu(1000000, 2.1, 16.0, seed=2); print("gen %.3f" % (time.time()-t))
plan = mb.QueryPlan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chi = np.stack([mb.random_coloring(g, 6, s) for s in range(100,108)])
import torch; torch.cuda.init(); torch.zeros(1, device='cuda'); torch.cuda.synchronize()
import os
os.environ["MB_DEBUG_PREP"]="1"
t=time.time(); c = mb.count_colorful(g, plan, chi); print("first call %.3f" % (time.time()-t), "prep_ms", mb.engine_prep_ms(g))
t=time.time(); c = mb.count_colorful(g, plan, chi); print("second call %.4f" % (time.time()-t))
e = g.edges(); n = g.num_vertices()
t=time.time(); g2 = mb.DataGraph.from_edges(n, e); print("from_edges %.3f" % (time.time()-t))
t=time.time(); c = mb.count_colorful(g2, plan, chi); print("first call on g2 %.3f" % (time.time()-t), "prep_ms", mb.engine_prep_ms(g2))
