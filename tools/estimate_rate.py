# estimate() end to end on the config-1 graph: trials/s with the colourings generated on the device
import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
g = mb.DataGraph.chung_lu(1000000, 2.1, 16.0, seed=2)
plan = mb.QueryPlan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
mb.estimate(g, plan, mb.DB, 8, 1)  # warm: upload + indexes
mb.engine_enable_timing(g, True)
for trials in (64, 256, 1024):
    t = time.time(); rep = mb.estimate(g, plan, mb.DB, trials, 7); dt = time.time() - t
    print(f"estimate: {trials} trials in {dt*1e3:.1f} ms = {trials/dt:.0f} trials/s  (mean {rep.mean_estimate:.6e}, cv {rep.cv:.4f})", flush=True)
for name, ms, n, b in mb.engine_timings(g):
    if name in ("random_colorings", "tri_hist_fused", "leaf_map", "recolor"): print(f"  {name:20s} {ms:10.3f} ms  {n:5d} launches")
t = time.time(); chis = np.stack([mb.random_coloring(g, 6, mb.derive_seed(7, i)) for i in range(64)]); dt = time.time() - t
print(f"host generation of 64 colourings (one thread): {dt*1e3:.1f} ms")
