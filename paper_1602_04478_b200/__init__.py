"""B200-native colour-coding engine for treewidth-2 subgraph counting.

Python mirror of the reference artifact's public API (C++ namespace ``motif``,
/root/reference/proj/include/motif/*.hpp) over the C ABI of
``libmotif_b200.so`` (declared in include/motif_b200.h).  Names, argument
meaning and error behaviour follow the reference:

=============================  ===============================================
here                           reference
=============================  ===============================================
``DataGraph.from_edges``       ``DataGraph::from_edges``        graph.hpp:20
``load_edge_list``             ``load_edge_list_file``          graph.hpp:48
``degree_rank``                ``degree_rank``                  graph.hpp:68
``random_coloring``            ``random_coloring``              graph.hpp:85
``QueryPlan``                  ``QueryGraph`` + ``enumerate_trees`` +
                               ``select_plan``                  query.hpp:25-108
``count_colorful``             ``count_colorful``               engine.hpp:121
``estimate``                   ``estimate``                     estimate.hpp:34
``automorphism_count``         ``automorphism_count``           estimate.hpp:14
``normalization_factor``       ``normalization_factor``         estimate.hpp:18
``Partition``                  ``Partition``                    runtime.hpp:14
=============================  ===============================================

There is no CPU fallback: importing this module loads the CUDA library and
fails loudly when it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MB_LIB_PATH: a developer override (an alternative in-tree build of the same
# library, e.g. a tuning variant from tools/build_variant.sh)
LIB_PATH = os.environ.get("MB_LIB_PATH") or os.path.join(_HERE, "libmotif_b200.so")

__all__ = [
    "MotifError", "ParseError", "TreewidthError", "CountOverflowError", "BudgetError",
    "SchemaError", "ContractError", "SpecError", "CudaError",
    "DataGraph", "QueryPlan", "EstimateReport", "Partition", "load_edge_list", "degree_rank",
    "random_coloring", "derive_seed", "count_colorful", "count_colorful_shard", "count_colorful_sharded", "device_random_colorings", "estimate", "automorphism_count",
    "normalization_factor", "coefficient_of_variation", "estimate_from_counts", "PS", "DB", "lib",
]

PS, DB = 0, 1


class MotifError(RuntimeError):
    code = 1


class ParseError(MotifError):
    code = 2


class TreewidthError(MotifError):
    code = 3


class CountOverflowError(MotifError):
    code = 4


class BudgetError(MotifError):
    code = 5


class SchemaError(MotifError):
    code = 6


class ContractError(MotifError):
    code = 7


class SpecError(MotifError):
    code = 8


class CudaError(MotifError):
    code = 9


_ERRORS = {c.code: c for c in (ParseError, TreewidthError, CountOverflowError, BudgetError,
                                SchemaError, ContractError, SpecError, CudaError)}


# mb_allgather_fn (include/motif_b200.h): int (*)(void* ctx, void* dev_buf, uint64_t bytes_per_rank, void* stream)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    u32p, u64p, i32p, u8p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                             C.POINTER(C.c_uint8))
    sig = {
        "mb_last_error": (C.c_char_p, []),
        "mb_version": (C.c_char_p, []),
        "mb_graph_from_edges": (C.c_int, [C.c_uint32, u32p, u32p, C.c_uint64, C.POINTER(P), u64p, u64p]),
        "mb_graph_load_edge_list": (C.c_int, [C.c_char_p, C.POINTER(P), u64p, u64p]),
        "mb_graph_gen_erdos_renyi": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(P)]),
        "mb_graph_gen_chung_lu": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                            C.POINTER(P)]),
        "mb_graph_gen_rmat": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                        C.POINTER(P)]),
        "mb_graph_free": (None, [P]),
        "mb_graph_num_vertices": (C.c_uint32, [P]),
        "mb_graph_num_edges": (C.c_uint64, [P]),
        "mb_graph_csr": (C.c_int, [P, u64p, u32p]),
        "mb_graph_edges": (C.c_int, [P, u32p, u32p]),
        "mb_graph_degree_rank": (C.c_int, [P, u32p]),
        "mb_graph_validate": (C.c_int, [P]),
        "mb_random_coloring": (C.c_int, [C.c_uint32, C.c_int, C.c_uint64, u8p]),
        "mb_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "mb_plan_create": (C.c_int, [C.c_int, i32p, C.c_int, C.c_uint64, C.POINTER(P)]),
        "mb_plan_load_query": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(P)]),
        "mb_plan_free": (None, [P]),
        "mb_plan_k": (C.c_int, [P]),
        "mb_plan_num_trees": (C.c_int, [P]),
        "mb_plan_selected": (C.c_int, [P]),
        "mb_plan_use_tree": (C.c_int, [P, C.c_int]),
        "mb_plan_canonical": (C.c_int, [P, C.c_int, C.c_char_p, C.c_int]),
        "mb_plan_score": (C.c_int, [P, C.c_int, C.POINTER(C.c_int)]),
        "mb_count_colorful": (C.c_int, [P, P, u8p, C.c_int, C.c_int, u64p]),
        "mb_count_colorful_seeds": (C.c_int, [P, P, u64p, C.c_int, C.c_int, u64p]),
        "mb_count_colorful_device": (C.c_int, [P, P, C.c_void_p, C.c_int, u64p]),
        "mb_device_random_colorings": (C.c_int, [P, C.c_int, u64p, C.c_int, C.c_uint64, u8p]),
        "mb_count_colorful_shard": (C.c_int, [P, P, u8p, C.c_int, C.c_int, C.c_int, C.c_int, u64p,
                                              C.POINTER(C.c_int)]),
        "mb_count_colorful_sharded": (C.c_int, [P, P, u8p, C.c_int, C.c_int, C.c_int, C.c_int, ALLGATHER_FN,
                                                C.c_void_p, u64p, C.POINTER(C.c_int)]),
        "mb_automorphism_count": (C.c_int, [C.c_int, i32p, C.c_int, u64p]),
        "mb_normalization_factor": (C.c_double, [C.c_int]),
        "mb_coefficient_of_variation": (C.c_double, [u64p, C.c_uint64]),
        "mb_estimate_from_counts": (C.c_int, [C.c_int, C.c_uint64, u64p, C.c_uint64, C.POINTER(C.c_double),
                                              C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "mb_estimate": (C.c_int, [P, P, C.c_int, C.c_uint64, C.c_uint64, u64p, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), u64p, C.POINTER(C.c_double)]),
        "mb_partition_block": (C.c_int, [C.c_uint32, C.c_int, C.c_int, u32p, u32p]),
        "mb_partition_owner": (C.c_int, [C.c_uint32, C.c_int, C.c_uint32, C.POINTER(C.c_int)]),
        "mb_engine_enable_timing": (C.c_int, [P, C.c_int]),
        "mb_engine_kernel_timing": (C.c_int, [P, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_double), u64p,
                                              u64p]),
        "mb_engine_stream": (C.c_void_p, [P]),
        "mb_engine_device": (C.c_int, [P]),
        "mb_engine_prep_ms": (C.c_double, [P]),
        "mb_engine_launches": (C.c_uint64, [P]),
        "mb_engine_exchanged_bytes": (C.c_uint64, [P]),
        "mb_engine_stats": (C.c_int, [P, u64p, u64p, u64p]),
        "mb_engine_reset_derived": (C.c_int, [P]),
        "mb_engine_release": (C.c_int, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.mb_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, MotifError)(msg)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class DataGraph:
    """Undirected simple graph in CSR form (reference graph.hpp:14)."""

    def __init__(self, handle: C.c_void_p, loops: int = 0, dups: int = 0):
        self._h = handle
        self.self_loops_dropped = loops
        self.duplicates_dropped = dups

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.mb_graph_free(h)
            self._h = None

    @classmethod
    def from_edges(cls, n: int, edges) -> "DataGraph":
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if e.size and (e.min() < 0 or e.max() >= n):
            raise SpecError("edge endpoint out of range")
        eu = np.ascontiguousarray(e[:, 0], dtype=np.uint32)
        ev = np.ascontiguousarray(e[:, 1], dtype=np.uint32)
        h = C.c_void_p()
        loops, dups = C.c_uint64(), C.c_uint64()
        _check(lib.mb_graph_from_edges(n, _ptr(eu, C.c_uint32), _ptr(ev, C.c_uint32), len(eu), C.byref(h),
                                       C.byref(loops), C.byref(dups)))
        return cls(h, loops.value, dups.value)

    @classmethod
    def erdos_renyi(cls, n: int, m: int, seed: int) -> "DataGraph":
        h = C.c_void_p()
        _check(lib.mb_graph_gen_erdos_renyi(n, m, seed, C.byref(h)))
        return cls(h)

    @classmethod
    def chung_lu(cls, n: int, gamma: float, avg_degree: float, seed: int, max_w: float = 0.0) -> "DataGraph":
        h = C.c_void_p()
        _check(lib.mb_graph_gen_chung_lu(n, gamma, avg_degree, max_w, seed, C.byref(h)))
        return cls(h)

    @classmethod
    def rmat(cls, scale: int, edge_factor: int, a: float, b: float, c: float, seed: int) -> "DataGraph":
        h = C.c_void_p()
        _check(lib.mb_graph_gen_rmat(scale, edge_factor, a, b, c, seed, C.byref(h)))
        return cls(h)

    @property
    def handle(self):
        return self._h

    def num_vertices(self) -> int:
        return lib.mb_graph_num_vertices(self._h)

    def num_edges(self) -> int:
        return lib.mb_graph_num_edges(self._h)

    def csr(self):
        n = self.num_vertices()
        off = np.empty(n + 1, dtype=np.uint64)
        adj = np.empty(max(2 * self.num_edges(), 1), dtype=np.uint32)
        _check(lib.mb_graph_csr(self._h, _ptr(off, C.c_uint64), _ptr(adj, C.c_uint32)))
        return off, adj[: 2 * self.num_edges()]

    def edges(self) -> np.ndarray:
        m = self.num_edges()
        eu = np.empty(max(m, 1), dtype=np.uint32)
        ev = np.empty(max(m, 1), dtype=np.uint32)
        _check(lib.mb_graph_edges(self._h, _ptr(eu, C.c_uint32), _ptr(ev, C.c_uint32)))
        return np.stack([eu[:m], ev[:m]], axis=1)

    def degree(self, v: int) -> int:
        off, _ = self.csr()
        return int(off[v + 1] - off[v])

    def validate(self) -> None:
        _check(lib.mb_graph_validate(self._h))

    def release_device(self) -> None:
        _check(lib.mb_engine_release(self._h))


def load_edge_list(path: str) -> DataGraph:
    h = C.c_void_p()
    loops, dups = C.c_uint64(), C.c_uint64()
    _check(lib.mb_graph_load_edge_list(path.encode(), C.byref(h), C.byref(loops), C.byref(dups)))
    return DataGraph(h, loops.value, dups.value)


def degree_rank(g: DataGraph) -> np.ndarray:
    r = np.empty(max(g.num_vertices(), 1), dtype=np.uint32)
    _check(lib.mb_graph_degree_rank(g.handle, _ptr(r, C.c_uint32)))
    return r[: g.num_vertices()]


def random_coloring(n_or_graph, k: int, seed: int) -> np.ndarray:
    n = n_or_graph.num_vertices() if isinstance(n_or_graph, DataGraph) else int(n_or_graph)
    chi = np.empty(max(n, 1), dtype=np.uint8)
    _check(lib.mb_random_coloring(n, k, seed, _ptr(chi, C.c_uint8)))
    return chi[:n]


def derive_seed(master: int, stream: int) -> int:
    return lib.mb_derive_seed(master, stream)


class QueryPlan:
    """Query graph + all decomposition trees + the §6-selected plan."""

    def __init__(self, k: int, edges: Sequence[tuple[int, int]], max_trees: int = 10000):
        e = np.asarray(list(edges), dtype=np.int32).reshape(-1, 2)
        h = C.c_void_p()
        _check(lib.mb_plan_create(k, _ptr(np.ascontiguousarray(e), C.c_int32), len(e), max_trees, C.byref(h)))
        self._h = h
        self.k = k
        self.edges = [tuple(map(int, x)) for x in e]

    @classmethod
    def from_file(cls, path: str, max_trees: int = 10000) -> "QueryPlan":
        obj = cls.__new__(cls)
        h = C.c_void_p()
        _check(lib.mb_plan_load_query(path.encode(), max_trees, C.byref(h)))
        obj._h = h
        obj.k = lib.mb_plan_k(h)
        obj.edges = []
        return obj

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.mb_plan_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def num_trees(self) -> int:
        return lib.mb_plan_num_trees(self._h)

    def selected(self) -> int:
        return lib.mb_plan_selected(self._h)

    def use_tree(self, idx: int) -> None:
        _check(lib.mb_plan_use_tree(self._h, idx))

    def canonical(self, idx: int = -1) -> str:
        buf = C.create_string_buffer(1 << 16)
        _check(lib.mb_plan_canonical(self._h, idx, buf, len(buf)))
        return buf.value.decode()

    def score(self, idx: int = -1) -> tuple[int, int, int]:
        s = (C.c_int * 3)()
        _check(lib.mb_plan_score(self._h, idx, s))
        return (s[0], s[1], s[2])


def count_colorful(g: DataGraph, plan: QueryPlan, chi: np.ndarray, engine: int = DB) -> int | np.ndarray:
    """Colourful matches (reference count_colorful, engine.hpp:121).

    ``chi`` is one colouring (n,) or a batch (c, n) with colours 1..k; a
    batch returns one count per colouring.
    """
    a = np.ascontiguousarray(chi, dtype=np.uint8)
    single = a.ndim == 1
    a2 = a.reshape(1, -1) if single else a
    if a2.shape[1] != g.num_vertices():
        raise SpecError("colouring length != number of vertices")
    out = np.zeros(a2.shape[0], dtype=np.uint64)
    _check(lib.mb_count_colorful(g.handle, plan.handle, _ptr(a2, C.c_uint8), a2.shape[0], engine,
                                 _ptr(out, C.c_uint64)))
    return int(out[0]) if single else out


def count_colorful_seeds(g: DataGraph, plan: QueryPlan, seeds: Iterable[int], engine: int = DB) -> np.ndarray:
    s = np.ascontiguousarray(list(seeds), dtype=np.uint64)
    out = np.zeros(len(s), dtype=np.uint64)
    _check(lib.mb_count_colorful_seeds(g.handle, plan.handle, _ptr(s, C.c_uint64), len(s), engine,
                                       _ptr(out, C.c_uint64)))
    return out


def device_random_colorings(g: DataGraph, k: int, seeds: Iterable[int], limit: int = 0) -> np.ndarray:
    """random_coloring(n, k, seed) of every seed as the device generates them
    for count_colorful_seeds / estimate (mb_device_random_colorings); (len(seeds), n)."""
    s = np.ascontiguousarray(list(seeds), dtype=np.uint64)
    out = np.zeros((len(s), g.num_vertices()), dtype=np.uint8)
    _check(lib.mb_device_random_colorings(g.handle, k, _ptr(s, C.c_uint64), len(s), limit, _ptr(out, C.c_uint8)))
    return out


def count_colorful_shard(g: DataGraph, plan: QueryPlan, chi: np.ndarray, rank: int, world: int,
                         engine: int = DB) -> tuple[np.ndarray, bool]:
    """This rank's partial counts of a vertex-sharded count (one per colouring)
    and whether the root block was split; partials of all ranks add up to
    count_colorful's counts (mb_count_colorful_shard)."""
    a = np.ascontiguousarray(np.atleast_2d(chi), dtype=np.uint8)
    if a.shape[1] != g.num_vertices():
        raise SpecError("colouring length != number of vertices")
    out = np.zeros(a.shape[0], dtype=np.uint64)
    split = C.c_int()
    _check(lib.mb_count_colorful_shard(g.handle, plan.handle, _ptr(a, C.c_uint8), a.shape[0], engine, rank, world,
                                       _ptr(out, C.c_uint64), C.byref(split)))
    return out, bool(split.value)


def count_colorful_sharded(g: DataGraph, plan: QueryPlan, chi: np.ndarray, rank: int, world: int, allgather,
                           engine: int = DB) -> tuple[np.ndarray, bool]:
    """mb_count_colorful_sharded: this rank's partial counts with the leaf
    blocks computed for its own vertices and their rows exchanged through
    ``allgather(dev_ptr, bytes_per_rank, cuda_stream)`` (an in-place all-gather
    over a device buffer of ``world`` slices, in stream order on the engine's
    stream; see parallel.make_allgather)."""
    a = np.ascontiguousarray(np.atleast_2d(chi), dtype=np.uint8)
    if a.shape[1] != g.num_vertices():
        raise SpecError("colouring length != number of vertices")
    out = np.zeros(a.shape[0], dtype=np.uint64)
    split = C.c_int()
    failure: list[BaseException] = []

    def _cb(_ctx, ptr, nbytes, stream):
        try:
            allgather(int(ptr), int(nbytes), int(stream or 0))
            return 0
        except BaseException as e:  # surfaces as CudaError below, with the cause attached
            failure.append(e)
            return 1

    cb = ALLGATHER_FN(_cb)
    try:
        _check(lib.mb_count_colorful_sharded(g.handle, plan.handle, _ptr(a, C.c_uint8), a.shape[0], engine, rank,
                                             world, cb, None, _ptr(out, C.c_uint64), C.byref(split)))
    except MotifError as e:
        if failure:
            raise e from failure[0]
        raise
    return out, bool(split.value)


def count_colorful_device(g: DataGraph, plan: QueryPlan, chi_dev_ptr: int, ncol: int) -> np.ndarray:
    out = np.zeros(ncol, dtype=np.uint64)
    _check(lib.mb_count_colorful_device(g.handle, plan.handle, C.c_void_p(chi_dev_ptr), ncol,
                                        _ptr(out, C.c_uint64)))
    return out


def automorphism_count(k: int, edges) -> int:
    e = np.ascontiguousarray(np.asarray(list(edges), dtype=np.int32).reshape(-1, 2))
    out = C.c_uint64()
    _check(lib.mb_automorphism_count(k, _ptr(e, C.c_int32), len(e), C.byref(out)))
    return out.value


def normalization_factor(k: int) -> float:
    if k < 1 or k > 32:
        raise SpecError("k out of range")
    return lib.mb_normalization_factor(k)


def coefficient_of_variation(counts) -> float:
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    return lib.mb_coefficient_of_variation(_ptr(c, C.c_uint64), len(c))


@dataclass
class EstimateReport:
    trials: int
    per_trial_colorful: list = field(default_factory=list)
    normalizer: float = 0.0
    mean_estimate: float = 0.0
    cv: float = 0.0
    aut: int = 0
    subgraph_estimate: float = 0.0


def estimate(g: DataGraph, plan: QueryPlan, engine: int, trials: int, seed: int) -> EstimateReport:
    per = np.zeros(max(trials, 1), dtype=np.uint64)
    mean, cv, sub = C.c_double(), C.c_double(), C.c_double()
    aut = C.c_uint64()
    _check(lib.mb_estimate(g.handle, plan.handle, engine, trials, seed, _ptr(per, C.c_uint64), C.byref(mean),
                           C.byref(cv), C.byref(aut), C.byref(sub)))
    return EstimateReport(trials, [int(x) for x in per[:trials]], normalization_factor(plan.k), mean.value,
                          cv.value, aut.value, sub.value)


def estimate_from_counts(k: int, edges, per_trial) -> EstimateReport:
    """estimate()'s report (estimate.cpp:124-129) from per-trial colourful
    counts computed elsewhere (the sharded multi-rank estimate): the mean is
    taken in long double by the library, as the reference does."""
    per = np.ascontiguousarray(per_trial, dtype=np.uint64)
    if len(per) < 1:
        raise SpecError("trials must be >= 1")
    aut = automorphism_count(k, edges)
    mean, cv, sub = C.c_double(), C.c_double(), C.c_double()
    _check(lib.mb_estimate_from_counts(k, aut, _ptr(per, C.c_uint64), len(per), C.byref(mean), C.byref(cv),
                                       C.byref(sub)))
    return EstimateReport(len(per), [int(x) for x in per], normalization_factor(k), mean.value, cv.value, aut,
                          sub.value)


class Partition:
    """1-D block distribution of vertices over p workers (runtime.hpp:14)."""

    def __init__(self, n: int, p: int):
        b, s = C.c_uint32(), C.c_uint32()
        _check(lib.mb_partition_block(n, p, 0, C.byref(b), C.byref(s)))
        self.n, self.p = n, p

    def workers(self) -> int:
        return self.p

    def block_begin(self, w: int) -> int:
        b, s = C.c_uint32(), C.c_uint32()
        _check(lib.mb_partition_block(self.n, self.p, w, C.byref(b), C.byref(s)))
        return b.value

    def block_size(self, w: int) -> int:
        b, s = C.c_uint32(), C.c_uint32()
        _check(lib.mb_partition_block(self.n, self.p, w, C.byref(b), C.byref(s)))
        return s.value

    def owner(self, v: int) -> int:
        o = C.c_int()
        _check(lib.mb_partition_owner(self.n, self.p, v, C.byref(o)))
        return o.value


def engine_timings(g: DataGraph) -> list[tuple[str, float, int, int]]:
    """(kernel name, summed device ms, launches, summed compulsory bytes)."""
    out = []
    i = 0
    buf = C.create_string_buffer(128)
    while True:
        ms, n, b = C.c_double(), C.c_uint64(), C.c_uint64()
        if lib.mb_engine_kernel_timing(g.handle, i, buf, 128, C.byref(ms), C.byref(n), C.byref(b)) != 0:
            break
        out.append((buf.value.decode(), ms.value, n.value, b.value))
        i += 1
    return out


def engine_enable_timing(g: DataGraph, on: bool = True) -> None:
    _check(lib.mb_engine_enable_timing(g.handle, 1 if on else 0))


def engine_device(g: DataGraph) -> int:
    """CUDA device the graph's engine runs on (-1 before the first count)."""
    return lib.mb_engine_device(g.handle)


def engine_stream(g: DataGraph) -> int:
    return lib.mb_engine_stream(g.handle) or 0


def engine_launches(g: DataGraph) -> int:
    return lib.mb_engine_launches(g.handle)


def engine_exchanged_bytes(g: DataGraph) -> int:
    """Bytes this rank received through count_colorful_sharded's exchanges."""
    return lib.mb_engine_exchanged_bytes(g.handle)


def engine_prep_ms(g: DataGraph) -> float:
    return lib.mb_engine_prep_ms(g.handle)


def engine_reset_derived(g: DataGraph) -> None:
    _check(lib.mb_engine_reset_derived(g.handle))


def engine_stats(g: DataGraph) -> dict:
    t, b, u = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(lib.mb_engine_stats(g.handle, C.byref(t), C.byref(b), C.byref(u)))
    return {"triangles": t.value, "table_bytes": b.value, "dp_updates": u.value}
