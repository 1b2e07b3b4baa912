#!/usr/bin/env python
"""Benchmark: colour-coding colourful-match counting on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

A *step* is one pass of the counting path over one batch of colourings of the
benchmark workload (config 1 by default: Chung-Lu n=1,000,000, exponent 2.1,
average degree 16, max expected degree sqrt(2m), graph seed 2; the 6-node
two-triangles-plus-pendant-path query; k=6; the batch = 8 colourings, seeds
100..107).  Graphs are seeded synthetic stand-ins (no datasets).

Our arm prints one JSON line with:
  value       colourings/s, graph + colourings resident in HBM, device-timed
              (CUDA events on the engine stream, max over ranks)
  e2e         colourings/s through the public C ABI (mb_count_colorful) with the
              colourings in pinned HOST memory, H2D/D2H inside the timed region
  roofline    dominant DP kernel: compulsory HBM bytes / its event-timed duration
  cpu_baseline the compiled reference (oracle/_ref) on a bounded sample of the
              same workload (same generator and query at reduced n), rank 0
  clocks      nvidia-smi samples during the timed region
Multi-GPU (torchrun): every rank counts its own batch of colourings (weak
scaling, no data-path collective); the device times are max-reduced over NCCL.

--impl reference runs the reference's own CPU implementation (oracle/_ref) on
all host threads on a bounded sample of the workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    0: dict(name="er10k_c5", gen=("er", 10_000, 50_000, 1), k=5,
            query=[(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)], seeds=[7], sample_n=10_000),
    1: dict(name="chunglu1m_tri2pendant_k6", gen=("cl", 1_000_000, 2.1, 16.0, 2), k=6,
            query=[(0, 1), (1, 2), (2, 0), (1, 3), (3, 2), (2, 4), (4, 5)], seeds=list(range(100, 108)),
            sample_n=20_000),
    2: dict(name="rmat22_c7", gen=("rmat", 22, 16, 3), k=7, query=[(i, (i + 1) % 7) for i in range(7)],
            seeds=list(range(200, 216)), sample_n=10, overflows=True),  # sample: R-MAT scale 10
    3: dict(name="chunglu4m_theta8", gen=("cl", 4_000_000, 2.3, 20.0, 4), k=8,
            query=[(0, 1), (1, 2), (2, 7), (0, 3), (3, 4), (4, 7), (0, 5), (5, 6), (6, 7)],
            seeds=list(range(300, 316)), sample_n=500),
    4: dict(name="chunglu2m_sp10", gen=("cl", 2_000_000, 2.1, 24.0, 5), k=10,
            query=[(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 2), (3, 5), (1, 6), (6, 7), (7, 8),
                   (8, 9), (9, 1), (1, 8)], seeds=list(range(400, 464)), sample_n=600, overflows=True),
}


def make_graph(mb, gen, n_override=None):
    kind = gen[0]
    if kind == "er":
        n, m, seed = gen[1:]
        if n_override:
            m = m * n_override // n
            n = n_override
        return mb.DataGraph.erdos_renyi(n, m, seed)
    if kind == "cl":
        n, gamma, avg, seed = gen[1:]
        return mb.DataGraph.chung_lu(n_override or n, gamma, avg, seed)
    scale, ef, seed = gen[1:]
    return mb.DataGraph.rmat(n_override or scale, ef, 0.57, 0.19, 0.19, seed)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def committed_limits(kernel: str):
    """ncu unit utilisations of the dominant kernel (profiles/r02_*_limits.json):
    which unit binds it when HBM does not."""
    p = os.path.join(ROOT, "profiles", f"r02_{kernel}_limits.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def committed_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(kernel)
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else None


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        # MB_BENCH_ONE_GPU=1 (tests on a one-GPU box): every rank on cuda:0,
        # gloo for the plumbing (NCCL refuses two ranks on one device)
        if os.environ.get("MB_BENCH_ONE_GPU"):
            backend, local = "gloo", 0
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def ref_layout(nc):
    """Host-thread layout for the reference: one colouring per thread (as its
    estimate() does, estimate.cpp:108-117), spare cores given to each colouring as
    BSP workers (parallel_count, runtime.cpp:311-324).  Measured on the 16-core GPU
    host at the config-1 sample: 8x1 0.60, 1x16 0.42, 8x2 0.69, 4x4 0.61 col/s."""
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    threads = max(1, min(ncpu, nc))
    return threads, max(1, ncpu // threads)


def sample_edges(cfg, n_override):
    """Edge list of the workload's bounded sample, generated by the product's
    seeded generator in a CHILD process and handed over as a .npy file, so the
    process that times the reference never maps libmotif_b200.so."""
    import tempfile

    gen = cfg["gen"]
    tag = "_".join(str(x) for x in gen) + f"_{n_override}"
    path = os.path.join(tempfile.gettempdir(), f"mb_sample_{tag}.npz")
    if not os.path.exists(path):
        code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
                "import paper_1602_04478_b200 as mb\n"
                "from bench import CONFIGS, make_graph\n"
                "g = make_graph(mb, CONFIGS[%d]['gen'], %r)\n"
                "np.savez(%r, n=g.num_vertices(), edges=g.edges())\n") % (ROOT, cfg["id"], n_override, path)
        subprocess.run([sys.executable, "-c", code], check=True)
    d = np.load(path)
    return int(d["n"]), d["edges"]


def time_reference(cfg, n_override, steps=1, warmup=0):
    """The compiled reference (oracle/_ref, DB engine, OpenMP) on the sample:
    one colouring per host thread, spare cores as BSP workers."""
    from oracle import Reference

    n, edges = sample_edges(cfg, n_override)
    R = Reference()
    rg = R.graph(n, edges)
    rp = R.plan(cfg["k"], cfg["query"])
    seeds = cfg["seeds"][:16]  # bounded sample: at most 16 colourings per step (one per host core)
    chis = np.stack([rg.coloring(cfg["k"], s) for s in seeds])
    threads, workers = ref_layout(len(chis))
    for _ in range(warmup):
        R.count_batch(rg, rp, chis[: min(len(chis), threads)], engine=1, threads=threads, workers=workers)
    t0 = time.perf_counter()
    for _ in range(steps):
        counts = R.count_batch(rg, rp, chis, engine=1, threads=threads, workers=workers)
    dt = (time.perf_counter() - t0) / steps
    return {"value": len(seeds) / dt, "dt": dt, "n": n, "m": len(edges), "colorings": len(seeds), "threads": threads,
            "workers": workers, "counts": [int(c) for c in counts], "seeds": seeds}


def reference_arm(args, cfg, ws, rank):
    if rank != 0:
        return
    r = time_reference(cfg, cfg["sample_n"], args.steps, args.warmup)
    v = r["value"]
    sample = (f"{cfg['name']} generator at n={r['n']} (m={r['m']}), same query/k/seeds; {r['colorings']} colourings "
              f"per step, {r['threads']} at a time x {r['workers']} BSP workers each")
    print(json.dumps({
        "impl": "reference", "metric": "colorings/sec", "value": v, "unit": "colorings/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["dt"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfg["name"], "sample_n": r["n"], "colorings_per_step": r["colorings"]},
        "cpu_baseline": {"value": v, "unit": "colorings/s", "cores": r["threads"] * r["workers"],
                         "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "colorings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "counts_first3": r["counts"][:3],
    }), flush=True)


def cpu_baseline(cfg):
    from oracle import reference_available

    if not reference_available() or not cfg["sample_n"]:
        return None
    r = time_reference(cfg, cfg["sample_n"])
    return {"value": r["value"], "unit": "colorings/s", "cores": r["threads"] * r["workers"], "kind": "reference",
            "counts": r["counts"],
            "sample": (f"compiled reference (oracle/_ref, DB engine) on the {cfg['name']} generator at "
                       f"n={r['n']} (m={r['m']}): {r['colorings']} colourings in {r['dt']:.1f}s, "
                       f"{r['threads']} colourings at a time x {r['workers']} BSP workers each")}


def gpu_rate(mb, g, plan, nb, chis_dev, pinned, steps, warmup, flush, dev):
    """Device-timed (CUDA events on the engine stream, L2 flushed between
    steps) and end-to-end (public C ABI, pinned host colourings, copies inside
    the region) colourings/s of one graph; returns counts too."""
    import torch

    stream = torch.cuda.ExternalStream(mb.engine_stream(g), device=dev)
    for _ in range(max(warmup, 0)):
        mb.count_colorful_device(g, plan, chis_dev.data_ptr(), nb)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        starts[i].record(stream)
        counts = mb.count_colorful_device(g, plan, chis_dev.data_ptr(), nb)
        ends[i].record(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in zip(starts, ends)]))
    t0 = time.perf_counter()
    for _ in range(steps):
        c = mb.count_colorful(g, plan, pinned.numpy())
    e2e_s = (time.perf_counter() - t0) / steps
    assert np.array_equal(c, counts)
    return ms, e2e_s, counts


def overflow_arm(args, cfg, ws, rank, local, g, plan, dev):
    """A workload whose colourful count is >= 2^64: the reference's checked
    u64 arithmetic raises OverflowError (errors.hpp:38-50), and so does the
    engine, failing fast at the first overflowing add.  A step resolves
    `per_step` colourings (one call each, as each would end the reference's
    estimate()); value = colourings resolved per second."""
    import torch

    import paper_1602_04478_b200 as mb

    k, n = cfg["k"], g.num_vertices()
    per_step = min(len(cfg["seeds"]), args.overflow_colorings)
    seeds = [s + rank * 1000 for s in cfg["seeds"][:per_step]]
    chis = [mb.random_coloring(g, k, s) for s in seeds]
    outcomes = []

    def step():
        res = []
        for chi in chis:
            try:
                res.append(int(mb.count_colorful(g, plan, chi)))
            except mb.CountOverflowError:
                res.append("OverflowError")
        return res

    t0 = time.perf_counter()
    outcomes = step()  # first call: upload + indexes
    first_call_s = time.perf_counter() - t0
    for _ in range(max(args.warmup - 1, 0)):
        step()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    clk = clocks.stop()
    t = torch.tensor([dt], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    dt = float(t.item())
    assert res == outcomes
    line = {
        "metric": "colorings/sec", "value": per_step * ws / dt, "unit": "colorings/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfg["name"] + (f"@size{args.size}" if args.size else ""), "n": n,
                   "m": g.num_edges(), "k": k, "colorings_per_step": per_step, "query_edges": cfg["query"],
                   "first_call_s": first_call_s,
                   "timing": "host wall clock around whole calls (each ends in an exception)"},
        "outcome": outcomes,
        "e2e": {"value": per_step * ws / dt, "unit": "colorings/s", "h2d_bytes_per_step": int(per_step * n),
                "d2h_bytes_per_step": int(8 * per_step)},
        "gpu_launches": None, "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def vertex_sharded_arm(args, cfg, ws, rank, local):
    """--sharding vertex: STRONG scaling of one batch — every rank takes its
    share of the data-graph vertices for the same colourings
    (mb_count_colorful_sharded: leaf rows exchanged with an all-gather per leaf
    table over NCCL, the root dealt over the ranks, partial counts all-gathered
    and added with checked u64 arithmetic).  Host wall clock around the whole
    call, max over ranks (the exchange runs on NCCL's stream)."""
    import torch

    import paper_1602_04478_b200 as mb
    from paper_1602_04478_b200 import parallel

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    g = make_graph(mb, cfg["gen"], args.size)
    plan = mb.QueryPlan(cfg["k"], cfg["query"])
    k, n, nb = cfg["k"], g.num_vertices(), len(cfg["seeds"])
    chis = np.stack([mb.random_coloring(g, k, s) for s in cfg["seeds"]])
    cdev = "cpu" if ws > 1 and torch.distributed.get_backend() != "nccl" else dev

    def step():
        return parallel.distributed_count_vertex_sharded(g, plan, chis, device=cdev, exchange=True)

    t0 = time.perf_counter()
    counts0 = step()
    first_call_s = time.perf_counter() - t0
    for _ in range(max(args.warmup - 1, 0)):
        step()
    x0 = mb.engine_exchanged_bytes(g)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        counts = step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    clk = clocks.stop()
    t = torch.tensor([dt], dtype=torch.float64, device=cdev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    dt = float(t.item())
    assert np.array_equal(counts, counts0)
    xb = (mb.engine_exchanged_bytes(g) - x0) // max(args.steps, 1)
    # the sharded totals against this rank's own unsharded count of the same batch
    whole = mb.count_colorful(g, plan, chis)
    if not np.array_equal(whole, counts0):
        raise SystemExit("bench: vertex-sharded counts differ from the unsharded count")
    line = {
        "metric": "colorings/sec", "value": nb / dt, "unit": "colorings/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfg["name"] + (f"@size{args.size}" if args.size else ""), "n": n, "m": g.num_edges(),
                   "k": k, "colorings_per_step": nb, "query_edges": cfg["query"],
                   "parallelism": f"vertices sharded over {ws} GPU(s), leaf rows exchanged",
                   "exchange_bytes_received_per_rank_per_step": int(xb), "first_call_s": first_call_s,
                   "timing": "host wall clock around whole calls, max over ranks"},
        "e2e": {"value": nb / dt, "unit": "colorings/s", "h2d_bytes_per_step": int(nb * n),
                "d2h_bytes_per_step": int(8 * nb)},
        "gpu_launches": None, "clocks": clk, "counts_first3": [int(x) for x in counts0[:3]],
        "counts_equal_unsharded": True,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def our_arm(args, cfg, ws, rank, local):
    import torch

    import paper_1602_04478_b200 as mb

    if args.sharding == "vertex":
        return vertex_sharded_arm(args, cfg, ws, rank, local)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    g = make_graph(mb, cfg["gen"], args.size)
    plan = mb.QueryPlan(cfg["k"], cfg["query"])
    k, n = cfg["k"], g.num_vertices()
    if cfg.get("overflows") and not args.size:
        return overflow_arm(args, cfg, ws, rank, local, g, plan, dev)
    # weak scaling: rank r counts its own batch (seed offset r * batch)
    nb = len(cfg["seeds"])
    seeds = [s + rank * 1000 for s in cfg["seeds"]]
    chis_host = np.stack([mb.random_coloring(g, k, s) for s in seeds])
    chis_dev = torch.from_numpy(chis_host).to(dev)
    pinned = torch.from_numpy(chis_host).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # first call: graph upload + plan-derived indexes + the count, from host
    # colourings (the cold end-to-end figure)
    t0 = time.perf_counter()
    counts0 = mb.count_colorful(g, plan, pinned.numpy())
    first_call_s = time.perf_counter() - t0
    prep_ms = mb.engine_prep_ms(g)
    assert mb.engine_device(g) == local, "engine not on this rank's device"
    stream = torch.cuda.ExternalStream(mb.engine_stream(g), device=dev)

    def step():
        return mb.count_colorful_device(g, plan, chis_dev.data_ptr(), nb)

    for _ in range(max(args.warmup, 0)):
        step()
    # timed region: K steps, barrier + synchronize on both sides, device events
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = mb.engine_launches(g)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    for i in range(args.steps):
        flush.zero_()  # L2 flush between steps (outside the event pair)
        torch.cuda.synchronize()
        starts[i].record(stream)
        counts = step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if ws > 1:
        torch.distributed.barrier()
    launches = (mb.engine_launches(g) - launches0) // max(args.steps, 1)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = float(np.mean(step_ms))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    value = nb * ws / (ms_max / 1e3)
    if not np.array_equal(counts, counts0):
        raise SystemExit("bench: counts changed between steps (nondeterminism)")

    # e2e: public C ABI with pinned HOST colourings, copies inside the region
    e2e_steps = max(args.steps, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        c = mb.count_colorful(g, plan, pinned.numpy())
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_value = nb * ws / float(te.item())
    assert np.array_equal(c, counts0)

    # seeds in, counts out: the colourings generated on the device (the path
    # estimate() takes), 256 seeds per call
    seed_list = [cfg["seeds"][0] + 1000 * (rank + 1) + i for i in range(256)]
    mb.count_colorful_seeds(g, plan, seed_list[:8])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cs = mb.count_colorful_seeds(g, plan, seed_list)
    seeds_s = time.perf_counter() - t0
    assert int(cs[0]) == int(mb.count_colorful(g, plan, mb.random_coloring(g, k, seed_list[0])))

    # roofline: one extra step with per-kernel CUDA-event timing
    mb.engine_enable_timing(g, True)
    step()
    timings = mb.engine_timings(g)
    mb.engine_enable_timing(g, False)
    dp = [t for t in timings if t[0].startswith(("leaf_", "tri_", "cycle_"))]
    total_dp_ms = sum(t[1] for t in dp)
    top = max(dp, key=lambda t: t[1])
    peaks = measured_peaks()
    per_launch_bytes = top[3] / max(top[2], 1)
    per_launch_ms = top[1] / max(top[2], 1)
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    stats = mb.engine_stats(g)
    line = {
        "metric": "colorings/sec", "value": value, "unit": "colorings/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfg["name"] + (f"@size{args.size}" if args.size else ""), "n": n, "m": g.num_edges(),
                   "k": k, "colorings_per_step": nb,
                   "query_edges": cfg["query"], "parallelism": f"colorings sharded over {ws} GPU(s)",
                   "l2": "flushed between steps (256 MB write) and working set > L2",
                   "graph_prep_ms": prep_ms, "first_call_s": first_call_s},
        "e2e": {"value": e2e_value, "unit": "colorings/s", "h2d_bytes_per_step": int(nb * n),
                "d2h_bytes_per_step": int(8 * nb + 24 * nb)},
        # cold end to end: a fresh graph handle's first call (graph upload,
        # degree-ordered relabel, common-neighbour index, the count)
        "e2e_cold": {"value": nb / first_call_s, "unit": "colorings/s", "seconds": first_call_s},
        # the seeded entry point (mb_count_colorful_seeds / mb_estimate): colourings
        # generated on the device, only seeds and counts cross PCIe
        "e2e_from_seeds": {"value": len(seed_list) / seeds_s, "unit": "colorings/s", "colorings": len(seed_list),
                           "h2d_bytes": 8 * len(seed_list), "d2h_bytes": 8 * len(seed_list)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": top[0], "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": committed_traffic(top[0]),
                     "algorithmic_bytes_per_launch": per_launch_bytes, "launch_ms": per_launch_ms,
                     "share_of_dp_time": top[1] / total_dp_ms if total_dp_ms else None,
                     "peak_source": peaks["source"], "ncu_limits": committed_limits(top[0])},
        "dp_table_updates_per_sec": stats["dp_updates"] / (ms_max / 1e3) * ws,
        "kernels": {t[0]: {"ms_per_step": t[1], "launches": t[2], "bytes": t[3]} for t in timings},
        "clocks": clk,
        "counts_first3": [int(x) for x in counts0[:3]],
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.size:
        cpu = cpu_baseline(cfg)
        line["cpu_baseline"] = cpu
        if cpu:
            # same input for both: the GPU on the reference's bounded sample
            gs = make_graph(mb, cfg["gen"], cfg["sample_n"])
            ss = cfg["seeds"][:16]
            cs = np.stack([mb.random_coloring(gs, k, s) for s in ss])
            cs_dev = torch.from_numpy(cs).to(dev)
            cs_pin = torch.from_numpy(cs).pin_memory()
            sms, se2e, scounts = gpu_rate(mb, gs, plan, len(ss), cs_dev, cs_pin, max(args.steps, 3), 2, flush, dev)
            same = [int(x) for x in scounts] == cpu["counts"]
            line["same_input"] = {
                "n": gs.num_vertices(), "m": gs.num_edges(), "colorings": len(ss),
                "value": len(ss) / (sms / 1e3), "e2e": len(ss) / se2e, "reference_value": cpu["value"],
                "ratio": len(ss) / (sms / 1e3) / cpu["value"], "e2e_ratio": len(ss) / se2e / cpu["value"],
                "counts_equal_reference": same, "same_config": True}
            if not same:
                raise SystemExit("bench: GPU counts differ from the reference on the same input")
        if cpu:
            cpu.pop("counts", None)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sample-n", type=int, default=None,
                    help="size of the bounded sample the reference (and the same-input GPU run) is timed on")
    ap.add_argument("--overflow-colorings", type=int, default=4,
                    help="colourings resolved per step on workloads whose count overflows u64 (configs 2, 4)")
    ap.add_argument("--sharding", choices=["colorings", "vertex"], default="colorings",
                    help="multi-GPU layout: colourings dealt over ranks (weak scaling, the default) or the "
                         "data-graph vertices of one batch sharded with leaf-row exchange (strong scaling)")
    ap.add_argument("--size", type=int, default=None,
                    help="override the generator size (n, or the R-MAT scale): supplementary reduced runs of "
                         "configs 2-4, whose full sizes exceed u64 counts or HBM (DESIGN.md)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], id=args.config)
    if args.sample_n:
        cfg["sample_n"] = args.sample_n
    ws, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            reference_arm(args, cfg, ws, rank)
        else:
            our_arm(args, cfg, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
