"""Generates the committed golden fixtures from the REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libmotif_ref.so, which is
compiled from /root/reference/proj/src by oracle/Makefile).  Outputs, all small
enough to commit:

  plans.json      canonical serialisation of every decomposition tree and of
                  the selected plan, plus plan scores, for a set of queries
                  (reference enumerate_trees / select_plan, query.cpp)
  colorings.json  reference random_coloring outputs (graph.cpp:142-151)
  counts.json     explicit small edge lists (seeded generators, frozen here as
                  edge lists), colouring seeds and the reference engine's
                  colourful counts (PS and DB, engine.cpp) for several queries
  estimates.json  reference estimate() per-trial counts / mean / cv

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402

QUERIES = {
    "edge": (2, [(0, 1)]),
    "p3": (3, [(0, 1), (1, 2)]),
    "p4": (4, [(0, 1), (1, 2), (2, 3)]),
    "star4": (5, [(0, 1), (0, 2), (0, 3), (0, 4)]),
    "c3": (3, [(0, 1), (1, 2), (2, 0)]),
    "c4": (4, [(0, 1), (1, 2), (2, 3), (3, 0)]),
    "c5": (5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)]),
    "c7": (7, [(i, (i + 1) % 7) for i in range(7)]),
    "q6": (6, [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2), (2, 4), (4, 5)]),
    "theta": (8, [(0, 1), (1, 2), (2, 7), (0, 3), (3, 4), (4, 7), (0, 5), (5, 6), (6, 7)]),
    # BASELINE config 4: 6-cycle with chords 0-2 and 3-5, path 1-6-7-8 and triangle 8-9-1 (14 edges)
    "sp10": (10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 2), (3, 5), (1, 6), (6, 7), (7, 8),
                  (8, 9), (9, 1), (1, 8)]),
    # the same without the chord 1-8 (a 5-cycle 1-6-7-8-9 instead of the triangle)
    "sp10_open": (10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 2), (3, 5), (1, 6), (6, 7), (7, 8),
                       (8, 9), (9, 1)]),
    "sat": (11, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (0, 5), (2, 6), (5, 6), (5, 7), (5, 8), (6, 8),
                 (8, 9), (9, 10), (10, 8)]),
    "brain1": (9, [(0, 1), (1, 2), (2, 3), (3, 0), (0, 4), (4, 5), (5, 6), (6, 7), (7, 8), (8, 0)]),
    "tri_pendant": (4, [(0, 1), (1, 2), (2, 3), (3, 1)]),
    "diamond": (4, [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2)]),
    "bowtie": (5, [(0, 1), (1, 2), (2, 0), (0, 3), (3, 4), (4, 0)]),
    "c5_pendant": (6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (2, 5)]),
}


def splitmix(x):
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


def er_edges(n, m, seed):
    """Frozen-here G(n, m): the list itself is the fixture."""
    seen, out, s = set(), [], seed
    while len(out) < m:
        s += 1
        u, v = splitmix(s) % n, splitmix(s ^ 0xABCDEF) % n
        if u == v:
            continue
        a, b = min(u, v), max(u, v)
        if (a, b) not in seen:
            seen.add((a, b))
            out.append((a, b))
    return out


def skewed_edges(n, m, seed):
    """Hub-heavy graph: endpoints drawn with weight ~ 1/(i+1)."""
    w = 1.0 / (np.arange(n) + 1.0)
    p = w / w.sum()
    rng = np.random.default_rng(seed)
    out, seen = [], set()
    while len(out) < m:
        u, v = rng.choice(n, 2, p=p)
        if u == v:
            continue
        a, b = int(min(u, v)), int(max(u, v))
        if (a, b) not in seen:
            seen.add((a, b))
            out.append((a, b))
    return out


def main():
    R = Reference()
    plans = {}
    for name, (k, q) in QUERIES.items():
        p = R.plan(k, q)
        plans[name] = {"k": k, "edges": q, "num_trees": p.num_trees(), "selected": p.canonical(-1),
                       "trees": [p.canonical(i) for i in range(p.num_trees())]}
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans, f, indent=1)

    g = R.graph(64, [(i, i + 1) for i in range(63)])
    colorings = {f"n64_k{k}_s{s}": [int(x) for x in g.coloring(k, s)] for k in (1, 3, 6, 10) for s in (0, 7, 100)}
    with open(os.path.join(HERE, "colorings.json"), "w") as f:
        json.dump(colorings, f)

    graphs = {
        "er24": (24, er_edges(24, 80, 11)),
        "er40": (40, er_edges(40, 110, 12)),
        "skew60": (60, skewed_edges(60, 200, 13)),
        "skew120": (120, skewed_edges(120, 420, 14)),
    }
    counts = {"graphs": {k: {"n": n, "edges": e} for k, (n, e) in graphs.items()}, "cases": []}
    for gname, (n, e) in graphs.items():
        rg = R.graph(n, e)
        for qname, (k, q) in QUERIES.items():
            if k >= 9 and n > 60:
                continue
            rp = R.plan(k, q)
            for seed in (1, 2):
                chi = rg.coloring(k, seed)
                ps = R.count(rg, rp, chi, engine=0)
                db = R.count(rg, rp, chi, engine=1)
                assert ps == db, (gname, qname, seed)
                counts["cases"].append({"graph": gname, "query": qname, "seed": seed, "colorful": db})
    with open(os.path.join(HERE, "counts.json"), "w") as f:
        json.dump(counts, f)

    est = []
    for gname in ("er24", "skew60"):
        n, e = graphs[gname]
        rg = R.graph(n, e)
        for qname in ("c3", "q6", "c5"):
            k, q = QUERIES[qname]
            per, mean, cv, sub = R.estimate(rg, R.plan(k, q), 1, 20, 77)
            est.append({"graph": gname, "query": qname, "trials": 20, "seed": 77,
                        "per_trial": [int(x) for x in per], "mean": mean, "cv": cv, "subgraph": sub})
    with open(os.path.join(HERE, "estimates.json"), "w") as f:
        json.dump(est, f, indent=1)
    print("golden fixtures written:", len(plans), "plans,", len(counts["cases"]), "count cases")


if __name__ == "__main__":
    main()
