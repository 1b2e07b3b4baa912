"""Pins BASELINE config 1 at FULL size with the independent OpenMP counter
(oracle/q6_count.c): Chung-Lu n=1,000,000, exponent 2.1, average degree 16,
graph seed 2, colouring seeds 100..107 -> tests/golden/config1_full.json.
The counter itself is checked against the compiled reference on the reduced
config-1 cases of tests/golden/configs.json (tests/test_oracle.py).

    python tools/pin_config1.py
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1602_04478_b200 as mb  # noqa: E402
from bench import CONFIGS  # noqa: E402
from oracle import Oracle  # noqa: E402

cfg = CONFIGS[1]
_, n, gamma, avg, gseed = cfg["gen"]
t0 = time.time()
g = mb.DataGraph.chung_lu(n, gamma, avg, gseed)
off, adj = g.csr()
sha = hashlib.sha1(g.edges().astype("<u4").tobytes()).hexdigest()
chis = np.stack([mb.random_coloring(g, cfg["k"], s) for s in cfg["seeds"]])
t1 = time.time()
counts = Oracle().q6_colorful(off, adj, chis)
t2 = time.time()
out = {"config": 1, "gen": list(cfg["gen"]), "n": g.num_vertices(), "m": g.num_edges(), "edges_sha1": sha,
       "k": cfg["k"], "query": cfg["query"], "seeds": cfg["seeds"], "colorful": counts,
       "counter": "oracle/q6_count.c (independent OpenMP counter, pinned against oracle/_ref)",
       "counter_seconds": round(t2 - t1, 2), "threads": os.cpu_count()}
print(json.dumps(out), f"graph {t1 - t0:.1f}s", flush=True)
with open(os.path.join(ROOT, "tests", "golden", "config1_full.json"), "w") as f:
    json.dump(out, f, indent=1)
