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
            seeds=list(range(200, 216)), sample_n=10),  # sample: R-MAT scale 10
    3: dict(name="chunglu4m_theta8", gen=("cl", 4_000_000, 2.3, 20.0, 4), k=8,
            query=[(0, 1), (1, 2), (2, 7), (0, 3), (3, 4), (4, 7), (0, 5), (5, 6), (6, 7)],
            seeds=list(range(300, 316)), sample_n=500),
    4: dict(name="chunglu2m_sp10", gen=("cl", 2_000_000, 2.1, 24.0, 5), k=10,
            query=[(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 2), (3, 5), (1, 6), (6, 7), (7, 8),
                   (8, 9), (9, 1)], seeds=list(range(400, 464)), sample_n=600),
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
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def ref_layout(nc):
    """Host-thread layout for the reference: one colouring per thread (as its
    estimate() does, estimate.cpp:149), spare cores given to each colouring as
    BSP workers (parallel_count, runtime.cpp:311).  Measured on the 16-core GPU
    host at the config-1 sample: 8x1 0.60, 1x16 0.42, 8x2 0.69, 4x4 0.61 col/s."""
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    threads = max(1, min(ncpu, nc))
    return threads, max(1, ncpu // threads)


def reference_arm(args, cfg, ws, rank):
    if rank != 0:
        return
    from oracle import Reference

    import paper_1602_04478_b200 as mb

    n_sample = cfg["sample_n"] or 10_000
    g = make_graph(mb, cfg["gen"], n_sample)
    R = Reference()
    rg = R.graph(g.num_vertices(), g.edges())
    rp = R.plan(cfg["k"], cfg["query"])
    seeds = cfg["seeds"][:16]  # bounded sample: at most 16 colourings per step (one per host core)
    chis = np.stack([rg.coloring(cfg["k"], s) for s in seeds])
    threads, workers = ref_layout(len(chis))
    for _ in range(args.warmup):
        R.count_batch(rg, rp, chis[: min(len(chis), threads)], engine=1, threads=threads, workers=workers)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        R.count_batch(rg, rp, chis, engine=1, threads=threads, workers=workers)
    dt = (time.perf_counter() - t0) / args.steps
    v = len(seeds) / dt
    sample = (f"{cfg['name']} generator at n={g.num_vertices()} (m={g.num_edges()}), same query/k/seeds; "
              f"{len(seeds)} colourings per step, {threads} at a time x {workers} BSP workers each")
    print(json.dumps({
        "impl": "reference", "metric": "colorings/sec", "value": v, "unit": "colorings/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfg["name"], "sample_n": g.num_vertices(), "colorings_per_step": len(seeds)},
        "cpu_baseline": {"value": v, "unit": "colorings/s", "cores": threads * workers,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "colorings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(cfg):
    from oracle import Reference, reference_available

    import paper_1602_04478_b200 as mb

    if not reference_available() or not cfg["sample_n"]:
        return None
    g = make_graph(mb, cfg["gen"], cfg["sample_n"])
    R = Reference()
    rg = R.graph(g.num_vertices(), g.edges())
    rp = R.plan(cfg["k"], cfg["query"])
    chis = np.stack([rg.coloring(cfg["k"], s) for s in cfg["seeds"][:16]])
    threads, workers = ref_layout(len(chis))
    t0 = time.perf_counter()
    R.count_batch(rg, rp, chis, engine=1, threads=threads, workers=workers)
    dt = time.perf_counter() - t0
    return {"value": len(chis) / dt, "unit": "colorings/s", "cores": threads * workers,
            "kind": "reference",
            "sample": (f"compiled reference (oracle/_ref, DB engine) on the {cfg['name']} generator at "
                       f"n={g.num_vertices()} (m={g.num_edges()}): {len(chis)} colourings in {dt:.1f}s, "
                       f"{threads} colourings at a time x {workers} BSP workers each")}


def our_arm(args, cfg, ws, rank, local):
    import torch

    import paper_1602_04478_b200 as mb

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    g = make_graph(mb, cfg["gen"], args.size)
    plan = mb.QueryPlan(cfg["k"], cfg["query"])
    k, n = cfg["k"], g.num_vertices()
    # weak scaling: rank r counts its own batch (seed offset r * batch)
    nb = len(cfg["seeds"])
    seeds = [s + rank * 1000 for s in cfg["seeds"]]
    chis_host = np.stack([mb.random_coloring(g, k, s) for s in seeds])
    chis_dev = torch.from_numpy(chis_host).to(dev)
    pinned = torch.from_numpy(chis_host).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # first call uploads the graph and builds the plan-derived indexes
    t0 = time.perf_counter()
    counts0 = mb.count_colorful_device(g, plan, chis_dev.data_ptr(), nb)
    first_call_s = time.perf_counter() - t0
    prep_ms = mb.engine_prep_ms(g)
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
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": top[0], "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": committed_traffic(top[0]),
                     "algorithmic_bytes_per_launch": per_launch_bytes, "launch_ms": per_launch_ms,
                     "share_of_dp_time": top[1] / total_dp_ms if total_dp_ms else None,
                     "peak_source": peaks["source"]},
        "dp_table_updates_per_sec": stats["dp_updates"] / (ms_max / 1e3) * ws,
        "kernels": {t[0]: {"ms_per_step": t[1], "launches": t[2], "bytes": t[3]} for t in timings},
        "clocks": clk,
        "counts_first3": [int(x) for x in counts0[:3]],
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
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
    ap.add_argument("--size", type=int, default=None,
                    help="override the generator size (n, or the R-MAT scale): supplementary reduced runs of "
                         "configs 2-4, whose full sizes exceed u64 counts or HBM (DESIGN.md)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
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
