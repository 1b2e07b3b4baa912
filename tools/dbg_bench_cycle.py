# device-timed (events on the engine stream, L2 flush between) vs e2e host loop for a cycle config
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1602_04478_b200 as mb
from bench import CONFIGS, make_graph
cfg = CONFIGS[int(sys.argv[1])]; size = int(sys.argv[2])
g = make_graph(mb, cfg["gen"], size)
plan = mb.QueryPlan(cfg["k"], cfg["query"])
chis = np.stack([mb.random_coloring(g, cfg["k"], s) for s in cfg["seeds"]])
dev = torch.device("cuda", 0)
chis_dev = torch.from_numpy(chis).to(dev)
nb = len(chis)
c0 = mb.count_colorful_device(g, plan, chis_dev.data_ptr(), nb)
stream = torch.cuda.ExternalStream(mb.engine_stream(g), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for mode in ("noflush", "flush", "noflush"):
    ts = []
    for i in range(3):
        if mode == "flush":
            flush.zero_()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record(stream); mb.count_colorful_device(g, plan, chis_dev.data_ptr(), nb); e.record(stream)
        torch.cuda.synchronize()
        ts.append((s.elapsed_time(e), (time.perf_counter() - t0) * 1e3))
    print(mode, [f"{a:.1f}/{b:.1f}" for a, b in ts], flush=True)
for i in range(3):
    t0 = time.perf_counter(); mb.count_colorful(g, plan, chis); print("e2e", f"{(time.perf_counter()-t0)*1e3:.1f} ms", flush=True)
