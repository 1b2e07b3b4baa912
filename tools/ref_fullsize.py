# Reference at the FULL config-1 size (n=1M), a few colourings, for DESIGN.md's
# honest full-size ratio (the bench's reference arm times a bounded n=20k sample).
import os, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
from oracle import Reference
nc = int(sys.argv[1]) if len(sys.argv) > 1 else 2
R = Reference()
g = mb.DataGraph.chung_lu(1_000_000, 2.1, 16.0, seed=2)
rg = R.graph(g.num_vertices(), g.edges())
rp = R.plan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chis = np.stack([mb.random_coloring(g, 6, s) for s in range(100, 100 + nc)])
ncpu = len(os.sched_getaffinity(0))
threads = nc
workers = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, ncpu // nc)
print("cpus", ncpu, "threads", threads, "workers", workers, flush=True)
t = time.time(); out = R.count_batch(rg, rp, chis, threads=threads, workers=workers); dt = time.time() - t
print(f"{nc} colourings in {dt:.1f}s -> {nc/dt:.5f} col/s", out.tolist(), flush=True)
