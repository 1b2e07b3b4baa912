# Timing split of the config-1 3-cycle kernel: MB_TRI_DEBUG=1 skips the join,
# 2 skips the list scan (counts are wrong in both; timing only).
import os, subprocess, sys
code = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
g = mb.DataGraph.chung_lu(1000000, 2.1, 16.0, seed=2)
plan = mb.QueryPlan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chi = np.stack([mb.random_coloring(g, 6, s) for s in range(100,108)])
mb.count_colorful(g, plan, chi)
mb.engine_enable_timing(g, True)
for _ in range(5): mb.count_colorful(g, plan, chi)
for name, ms, n, b in mb.engine_timings(g):
    if name.startswith('tri'): print(name, round(ms / 5, 4))
'''
for mode in sys.argv[1:] or ["0", "1", "2", "3"]:
    env = dict(os.environ, MB_TRI_DEBUG=mode)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("mode", mode, out.stdout.strip(), out.stderr.strip()[-300:])
