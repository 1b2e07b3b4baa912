import sys, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
from bench import CONFIGS, make_graph
cfg = CONFIGS[3]
g = make_graph(mb, cfg["gen"], int(sys.argv[1]))
plan = mb.QueryPlan(cfg["k"], cfg["query"])
chi = mb.random_coloring(g, cfg["k"], cfg["seeds"][0])
print(mb.count_colorful(g, plan, chi))
