# one colouring of a config at a given size, with per-kernel engine timings
#   python tools/dbg_cfg.py CONFIG SIZE [ncolourings]
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1602_04478_b200 as mb
from bench import CONFIGS, make_graph
cfg = CONFIGS[int(sys.argv[1])]
sz = int(sys.argv[2]); nc = int(sys.argv[3]) if len(sys.argv) > 3 else 1
gen = cfg["gen"]
g = mb.DataGraph.rmat(sz, gen[2], 0.57, 0.19, 0.19, gen[3]) if gen[0] == "rmat" else make_graph(mb, gen, sz)
plan = mb.QueryPlan(cfg["k"], cfg["query"])
print(plan.canonical(), "n", g.num_vertices(), "m", g.num_edges(), flush=True)
chi = np.stack([mb.random_coloring(g, cfg["k"], s) for s in cfg["seeds"][:nc]])
c = mb.count_colorful(g, plan, chi)
mb.lib.mb_engine_enable_timing(g.handle, 1)
t = time.time(); c = mb.count_colorful(g, plan, chi); dt = time.time() - t
print("count", c, f"{dt:.3f}s", "launches", mb.engine_launches(g), flush=True)
tot = 0
rows = sorted(mb.engine_timings(g), key=lambda r: -r[1])
for name, ms, l, b in rows: tot += ms
for name, ms, l, b in rows[:25]: print(f"  {name:24s} {ms:10.3f} ms {l:7d}  {ms/tot*100:5.1f}%")
print(f"  total kernel time {tot:.1f} ms of {dt*1e3:.1f} ms wall")
