"""Multi-GPU counting: one process per GPU.

Two shardings, both without a data-path collective:

* colourings (``distributed_count_seeds`` / ``distributed_estimate``): rank r
  counts the contiguous block of colourings that Partition(num_colourings,
  world).block(r) assigns it (runtime.hpp:14-36), each on its own GPU with the
  whole graph resident, and the per-colouring counts are all-gathered once at
  the end (NCCL on GPUs, gloo on CPU).  This is the layout for plans whose
  tables fit one GPU (configs 0 and 1) and for estimate()'s independent trials
  (estimate.cpp:108-117).
* vertices (``distributed_count_vertex_sharded``): one colouring's root block
  is split by anchor vertex, the data-graph vertices being dealt to ranks as
  the reference's Partition deals them to BSP workers (runtime.cpp:11-25, here
  cyclically over the degree order so every rank gets its share of hubs); each
  rank sums the matches anchored at its own vertices and the partial counts
  are added with one all-reduce (the reference's sharded total,
  runtime.cpp:297-302).  See DESIGN.md §6.

  With ``exchange=True`` the leaf blocks are sharded as well: every rank
  computes the rows of its own vertices and the rows are exchanged with an
  all-gather per leaf table (``make_allgather``: NCCL in place on the device
  buffer, or staged through the host for gloo) — the halo exchange the
  reference performs when redistribute / extend ship entries to the owner of
  their key vertex (runtime.cpp:94-114, 173-202) — and a root 3-cycle block
  is dealt over the ranks by warp batch of oriented edges
  (mb_count_colorful_sharded).

Results are bit-identical to the single-GPU call for every world size.
``count_fn`` lets the CPU tests drive the same plumbing with the oracle.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from . import EstimateReport, derive_seed, estimate_from_counts


def block(n: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of rank's block: Partition(n, p) (runtime.hpp:14-25);
    the first n % p ranks hold one extra item; empty blocks when n < p."""
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def _world():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_world_size(), dist.get_rank()
    return None, 1, 0


def _all_gather_counts(local: np.ndarray, total: int, dist, world: int, device) -> np.ndarray:
    import torch

    # pad every rank's block to the largest block, gather, then trim
    width = -(-total // world)
    buf = torch.zeros(width, dtype=torch.int64, device=device)
    if len(local):
        buf[: len(local)] = torch.from_numpy(local.astype(np.uint64).view(np.int64)).to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = []
    for r in range(world):
        b, e = block(total, world, r)
        out.append(parts[r][: e - b].cpu().numpy().view(np.uint64))
    return np.concatenate(out) if out else np.zeros(0, np.uint64)


def distributed_count_seeds(g, plan, seeds: Sequence[int], engine: int = 1,
                            count_fn: Callable | None = None, device=None) -> np.ndarray:
    """Colourful counts for the colourings random_coloring(n, k, seed) of every
    seed, computed across all ranks; every rank returns the full list."""
    from . import count_colorful_seeds

    dist, world, rank = _world()
    b, e = block(len(seeds), world, rank)
    mine = list(seeds[b:e])
    if count_fn is not None:
        local = np.asarray([count_fn(s) for s in mine], dtype=np.uint64)
    else:
        local = count_colorful_seeds(g, plan, mine, engine) if mine else np.zeros(0, np.uint64)
    if world == 1:
        return local
    if device is None:
        import torch

        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    return _all_gather_counts(local, len(seeds), dist, world, device)


def distributed_estimate(g, plan, engine: int, trials: int, seed: int, k: int | None = None,
                         edges=None, count_fn: Callable | None = None, device=None) -> EstimateReport:
    """estimate() (estimate.hpp:34) with the trials sharded over the ranks.
    Trial i uses derive_seed(seed, i) exactly as the single-process call, so
    the report is identical for every world size."""
    if trials < 1:
        raise ValueError("trials must be >= 1")
    k = plan.k if k is None else k
    edges = plan.edges if edges is None else edges
    seeds = [derive_seed(seed, i) for i in range(trials)]
    per = distributed_count_seeds(g, plan, seeds, engine, count_fn, device)
    return estimate_from_counts(k, edges, per)


def sum_partials(parts: Sequence[Sequence[int]], overflowed: Sequence[bool]) -> np.ndarray:
    """Adds the ranks' partial counts with the reference's checked u64
    arithmetic (errors.hpp:38-50): a rank that overflowed, or a sum >= 2^64,
    is the reference's OverflowError."""
    from . import CountOverflowError

    if any(overflowed):
        raise CountOverflowError("count overflow (64-bit)")
    tot = [sum(int(p[c]) for p in parts) for c in range(len(parts[0]))] if parts else []
    if any(t >= 1 << 64 for t in tot):
        raise CountOverflowError("count overflow in addition")
    return np.asarray(tot, dtype=np.uint64)


class _DeviceBytes:
    """A raw device allocation as a __cuda_array_interface__ object, so that
    torch can wrap the engine's exchange buffer without copying it."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 2}


def gather_slices(slices: Sequence[np.ndarray]) -> np.ndarray:
    """The exchange buffer after the all-gather: rank q's packed rows in slice
    q (host-side model of the layout, used by the CPU tests)."""
    return np.concatenate([np.asarray(s, dtype=np.uint8) for s in slices])


def make_allgather(dist, world: int, rank: int, device=None):
    """The ``allgather(dev_ptr, bytes_per_rank, cuda_stream)`` callback of
    count_colorful_sharded over torch.distributed: the engine has packed this
    rank's rows into slice ``rank`` of the device buffer (ready in stream order
    on its stream); on return every slice holds its rank's rows, again in
    stream order on that stream.  NCCL gathers in place on the device (NVLink)
    with the engine's stream current, so nothing blocks the host; other
    backends synchronise and stage the slices through host memory."""
    import torch

    nccl = dist.get_backend() == "nccl"
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    on_host = torch.device(device).type == "cpu"  # CPU tests: the buffer is host memory

    def allgather(ptr: int, nbytes: int, stream: int = 0) -> None:
        if on_host:
            import ctypes

            buf = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * (nbytes * world)).from_address(ptr)))
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, buf[rank * nbytes:(rank + 1) * nbytes].clone())
            buf.copy_(torch.from_numpy(gather_slices([p.numpy() for p in parts])))
            return
        ext = torch.cuda.ExternalStream(stream, device=device) if stream else torch.cuda.current_stream(device)
        with torch.cuda.stream(ext):
            buf = torch.as_tensor(_DeviceBytes(ptr, nbytes * world), device=device)
            mine = buf[rank * nbytes:(rank + 1) * nbytes]
            if nccl:
                # NCCL orders itself after the current stream (the engine's) and
                # the current stream after the collective: asynchronous
                dist.all_gather_into_tensor(buf, mine.clone())
            else:
                parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, mine.cpu())  # .cpu() waits for the packed rows
                buf.copy_(torch.from_numpy(gather_slices([p.numpy() for p in parts])))
                ext.synchronize()  # the staging tensor must outlive the copy

    return allgather


def distributed_count_vertex_sharded(g, plan, chis, engine: int = 1, count_fn: Callable | None = None,
                                     device=None, exchange: bool = False) -> np.ndarray:
    """Counts of the colourings `chis` (c, n) with the data-graph vertices
    sharded over the ranks: each rank sums the root-block matches anchored at
    its vertices (mb_count_colorful_shard), and the partials are combined by
    one all-gather + checked sum, the reference's sharded total
    (runtime.cpp:297-302).  Every rank returns the full counts.
    ``count_fn(rank, world) -> (partials, overflowed)`` replaces the device
    call in the CPU tests."""
    import torch

    from . import CountOverflowError, count_colorful_shard, count_colorful_sharded

    dist, world, rank = _world()
    chis = np.atleast_2d(chis)
    overflowed = False
    if count_fn is not None:
        part, overflowed = count_fn(rank, world)
        part = np.asarray(part, dtype=np.uint64)
    else:
        try:
            if exchange and world > 1:
                part, _ = count_colorful_sharded(g, plan, chis, rank, world, make_allgather(dist, world, rank), engine)
            else:
                part, _ = count_colorful_shard(g, plan, chis, rank, world, engine)
        except CountOverflowError:
            part, overflowed = np.zeros(len(chis), np.uint64), True
    if world == 1:
        return sum_partials([part], [overflowed])
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    buf = torch.zeros(len(chis) + 1, dtype=torch.int64, device=device)
    buf[: len(chis)] = torch.from_numpy(part.astype(np.uint64).view(np.int64)).to(device)
    buf[len(chis)] = 1 if overflowed else 0
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    rows = [t.cpu().numpy().view(np.uint64) for t in gathered]
    return sum_partials([r[:-1] for r in rows], [bool(r[-1]) for r in rows])
