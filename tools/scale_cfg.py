# time one colouring of a config's query on its generator at increasing sizes
#   python tools/scale_cfg.py CONFIG SIZE1 SIZE2 ...   (sizes: n, or R-MAT scale)
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1602_04478_b200 as mb
sys.path.insert(0, '.')
from bench import CONFIGS, make_graph
cfg = CONFIGS[int(sys.argv[1])]
for sz in sys.argv[2:]:
    sz = int(sz)
    gen = cfg["gen"]
    if gen[0] == "rmat":
        g = mb.DataGraph.rmat(sz, gen[2], 0.57, 0.19, 0.19, gen[3])
    else:
        g = make_graph(mb, gen, sz)
    plan = mb.QueryPlan(cfg["k"], cfg["query"])
    chi = np.stack([mb.random_coloring(g, cfg["k"], s) for s in cfg["seeds"][:1]])
    t = time.time()
    import os
    if os.environ.get("MB_TIMING"):
        try:
            mb.count_colorful(g, plan, mb.random_coloring(g, cfg["k"], 1))  # warm: upload + indexes
        except mb.CountOverflowError:
            pass
        mb.engine_enable_timing(g, True)
        t = time.time()
    try:
        c = mb.count_colorful(g, plan, chi)
        dt = time.time() - t
        t2 = time.time(); c2 = mb.count_colorful(g, plan, chi); dt2 = time.time() - t2
        print(f"size {sz} n={g.num_vertices()} m={g.num_edges()} first {dt:.3f}s again {dt2:.3f}s count {c[0]}",
              mb.engine_stats(g), flush=True)
    except Exception as e:
        print(f"size {sz} n={g.num_vertices()} m={g.num_edges()} FAILED after {time.time()-t:.1f}s: {e}", flush=True)
    if os.environ.get("MB_TIMING"):
        for name, ms, n, b in sorted(mb.engine_timings(g), key=lambda t: -t[1])[:12]:
            print(f"   {name:28s} {ms:10.2f} ms  {n:7d} launches  {b / max(ms, 1e-9) / 1e6:8.1f} GB/s", flush=True)
        mb.engine_enable_timing(g, False)
        continue
