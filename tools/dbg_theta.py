import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1602_04478_b200 as mb
from bench import CONFIGS, make_graph
cfg = CONFIGS[3]
n = int(sys.argv[1]); nc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = make_graph(mb, cfg["gen"], n)
plan = mb.QueryPlan(cfg["k"], cfg["query"])
print(plan.canonical(), flush=True)
chi = np.stack([mb.random_coloring(g, cfg["k"], s) for s in cfg["seeds"][:nc]])
t = time.time(); c = mb.count_colorful(g, plan, chi); print("count", c, time.time() - t, flush=True)
for name, ms, l, b in mb.engine_timings(g)[:30]: print(f"  {name:24s} {ms:10.3f} ms {l:6d}")
