# One rank's share of a vertex-sharded config-1 batch, measured on one GPU: rank 0 of W runs its
# leaf kernels on the vertices it owns and its share of the root kernel; the exchange callback does
# nothing (the other ranks' rows stay stale, so the partial count is meaningless — only the kernel
# times and the exchanged byte counts are read).  Projects the compute side of strong scaling.
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1602_04478_b200 as mb
g = mb.DataGraph.chung_lu(1000000, 2.1, 16.0, seed=2)
plan = mb.QueryPlan(6, [(0,1),(1,2),(2,0),(1,3),(3,2),(2,4),(4,5)])
chi = np.stack([mb.random_coloring(g, 6, s) for s in range(100, 108)])
mb.count_colorful(g, plan, chi)
for W in (1, 2, 4, 8):
    for rep in range(2):
        mb.engine_enable_timing(g, True)
        x0 = mb.engine_exchanged_bytes(g)
        if W == 1: mb.count_colorful(g, plan, chi)
        else: mb.count_colorful_sharded(g, plan, chi, 0, W, lambda ptr, nbytes, stream: None)
        t = {name: ms for name, ms, n, b in mb.engine_timings(g)}
        xb = mb.engine_exchanged_bytes(g) - x0
        mb.engine_enable_timing(g, False)
    leaf1 = max(t.get("leaf_hist", 0), t.get("leaf_hist_heavy", 0)); leaf2 = max(t.get("leaf_map", 0), t.get("leaf_map_heavy", 0))
    tri = t.get("tri_hist_fused", 0); pk = t.get("shard_pack", 0) + t.get("shard_unpack", 0)
    comp = leaf1 + leaf2 + tri + t.get("recolor", 0) + pk
    nvl = xb / 900e9 * 1e3
    print(f"W={W}: leaf level 1 {leaf1:.3f} ms, level 2 {leaf2:.3f} ms, root {tri:.3f} ms, pack+unpack {pk:.3f} ms, "
          f"compute {comp:.3f} ms; received {xb/1e6:.1f} MB = {nvl:.3f} ms at 900 GB/s; projected step {comp+nvl:.3f} ms", flush=True)
    print("     " + ", ".join(f"{k} {v:.3f}" for k, v in sorted(t.items())), flush=True)
