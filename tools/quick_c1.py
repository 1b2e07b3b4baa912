import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
t=time.time(); g = mb.DataGraph.chung_lu(1000000, 2.1, 16.0, seed=2); print("gen", time.time()-t, g.num_edges(), flush=True)
plan = mb.QueryPlan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chi = np.stack([mb.random_coloring(g, 6, s) for s in range(100,108)])
mb.engine_enable_timing(g, True) if False else None
c0 = mb.count_colorful(g, plan, chi); print("prep_ms", mb.engine_prep_ms(g), c0[:3])
mb.lib.mb_engine_enable_timing(g.handle, 1)
for rep in range(3):
    t=time.time(); c = mb.count_colorful(g, plan, chi); dt=time.time()-t
    print("rep", rep, dt, c[:3], mb.engine_stats(g), flush=True)
for name, ms, n, b in mb.engine_timings(g): print(f"  {name:20s} {ms:10.3f} ms  {n:5d}  {b/max(ms,1e-9)/1e6:10.1f} GB/s")
