# small end-to-end counts with every launch synchronised and checked (MB_SYNC_DEBUG=1), or under
# compute-sanitizer where the pool allows it:
#   compute-sanitizer --tool memcheck python tools/sanitize_small.py
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
g = mb.DataGraph.chung_lu(1500, 2.1, 10.0, 3)
qs = {"q6": (6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)]),
      "c5": (5, [(i, (i+1) % 5) for i in range(5)]),
      "theta": (8, [(0,1),(1,2),(2,7),(0,3),(3,4),(4,7),(0,5),(5,6),(6,7)]),
      "tri_tails": (6, [(0,1),(1,2),(2,0),(0,3),(1,4),(4,5)])}
for name, (k, q) in qs.items():
    plan = mb.QueryPlan(k, q)
    chis = np.stack([mb.random_coloring(g, k, s) for s in range(9)])
    print(name, [int(x) for x in mb.count_colorful(g, plan, chis)][:3])
    # one rank of a 2-rank sharded count with a no-op exchange (rows of the other rank stay stale:
    # the partial is meaningless, the kernels and index arithmetic are what is checked)
    try:
        mb.count_colorful_sharded(g, plan, chis, 1, 2, lambda ptr, nbytes, stream: None)
    except mb.MotifError as e:
        print("  sharded dry run:", type(e).__name__)
