# which host-thread layout runs the reference fastest on this box (config-1 sample)
import os, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
from oracle import Reference
R = Reference()
g = mb.DataGraph.chung_lu(20000, 2.1, 16.0, seed=2)
rg = R.graph(g.num_vertices(), g.edges())
rp = R.plan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chis = np.stack([mb.random_coloring(g, 6, s) for s in range(100, 108)])
ncpu = os.cpu_count()
print("cpus", ncpu, "affinity", len(os.sched_getaffinity(0)), flush=True)
for threads, workers in [(8, 1), (1, ncpu), (8, max(1, ncpu // 8)), (4, max(1, ncpu // 4))]:
    t = time.time(); out = R.count_batch(rg, rp, chis, threads=threads, workers=workers); dt = time.time() - t
    print(threads, workers, f"{dt:.2f}s", f"{8/dt:.3f} col/s", out[:2], flush=True)
