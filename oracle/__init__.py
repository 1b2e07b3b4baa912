"""TEST INFRASTRUCTURE ONLY — the CPU oracle and the compiled reference.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package; the
product (``paper_1602_04478_b200``) never does.

* ``Oracle``     — plain-C restatement (oracle/motif_oracle.c) of the
  reference's ground-truth path: mt19937_64 colourings, CSR normalisation,
  degree rank, brute-force colourful/match counting, automorphisms, k^k/k!,
  cv.  Each C function cites the reference file:line it restates.
* ``Reference``  — the unmodified reference library (oracle/_ref/libmotif_ref.so,
  compiled from /root/reference/proj/src by oracle/Makefile) behind a thin
  marshalling shim (oracle/ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libmotif_ref.so")

u8p, u32p, u64p, i32p = (C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                         C.POINTER(C.c_int32))


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = C.CDLL(path)
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64]
        L.or_derive_seed.restype = C.c_uint64
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_mt64_stream.argtypes = [C.c_uint64, C.c_uint64, u64p]
        L.or_random_coloring.restype = C.c_int
        L.or_random_coloring.argtypes = [C.c_uint32, C.c_int, C.c_uint64, u8p]
        L.or_build_csr.restype = C.c_uint64
        L.or_build_csr.argtypes = [C.c_uint32, u32p, u32p, C.c_uint64, u64p, u32p]
        L.or_degree_rank.argtypes = [C.c_uint32, u64p, u32p]
        L.or_brute_count.restype = C.c_int
        L.or_brute_count.argtypes = [C.c_uint32, u64p, u32p, u8p, C.c_int, i32p, C.c_int, C.c_uint64, u64p]
        L.or_automorphism_count.restype = C.c_int
        L.or_automorphism_count.argtypes = [C.c_int, i32p, C.c_int, u64p]
        L.or_normalization_factor.restype = C.c_double
        L.or_normalization_factor.argtypes = [C.c_int]
        L.or_coefficient_of_variation.restype = C.c_double
        L.or_coefficient_of_variation.argtypes = [u64p, C.c_uint64]
        L.or_q6_colorful.restype = C.c_int
        L.or_q6_colorful.argtypes = [C.c_uint32, u64p, u32p, C.c_int, u8p, u64p]
        self.L = L

    def mt64(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        self.L.or_mt64_stream(seed, count, _p(out, C.c_uint64))
        return out

    def derive_seed(self, master: int, stream: int) -> int:
        return self.L.or_derive_seed(master, stream)

    def random_coloring(self, n: int, k: int, seed: int) -> np.ndarray:
        chi = np.empty(max(n, 1), dtype=np.uint8)
        if self.L.or_random_coloring(n, k, seed, _p(chi, C.c_uint8)) != 0:
            raise OracleError(8, "k out of range")
        return chi[:n]

    def build_csr(self, n: int, edges):
        e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
        eu, ev = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
        off = np.zeros(n + 1, dtype=np.uint64)
        adj = np.zeros(max(2 * len(e), 1), dtype=np.uint32)
        m = self.L.or_build_csr(n, _p(eu, C.c_uint32), _p(ev, C.c_uint32), len(e), _p(off, C.c_uint64),
                                _p(adj, C.c_uint32))
        return off, adj[: 2 * m], m

    def degree_rank(self, off: np.ndarray) -> np.ndarray:
        n = len(off) - 1
        r = np.empty(max(n, 1), dtype=np.uint32)
        self.L.or_degree_rank(n, _p(np.ascontiguousarray(off, dtype=np.uint64), C.c_uint64), _p(r, C.c_uint32))
        return r[:n]

    def brute(self, off, adj, k, qedges, chi=None, budget=10**9) -> int:
        q = np.ascontiguousarray(np.asarray(qedges, dtype=np.int32).reshape(-1, 2))
        off = np.ascontiguousarray(off, dtype=np.uint64)
        adj = np.ascontiguousarray(adj if len(adj) else np.zeros(1), dtype=np.uint32)
        out = C.c_uint64()
        chip = None if chi is None else _p(np.ascontiguousarray(chi, dtype=np.uint8), C.c_uint8)
        rc = self.L.or_brute_count(len(off) - 1, _p(off, C.c_uint64), _p(adj, C.c_uint32), chip, k,
                                   _p(q, C.c_int32), len(q), budget, C.byref(out))
        if rc:
            raise OracleError(rc, "oracle budget exceeded")
        return out.value

    def q6_colorful(self, off, adj, chis) -> list:
        """Independent OpenMP counter of BASELINE config 1's query (q6_count.c)
        for a batch of colourings (c, n); raises on u64 overflow."""
        off = np.ascontiguousarray(off, dtype=np.uint64)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        chis = np.ascontiguousarray(np.atleast_2d(chis), dtype=np.uint8)
        out = np.zeros(chis.shape[0], dtype=np.uint64)
        rc = self.L.or_q6_colorful(len(off) - 1, _p(off, C.c_uint64), _p(adj, C.c_uint32), chis.shape[0],
                                   _p(chis, C.c_uint8), _p(out, C.c_uint64))
        if rc == -1:
            raise OracleError(4, "count overflow (64-bit)")
        if rc != 0:
            raise OracleError(8, f"q6 counter failed ({rc})")
        return [int(x) for x in out]

    def automorphism_count(self, k, qedges) -> int:
        q = np.ascontiguousarray(np.asarray(qedges, dtype=np.int32).reshape(-1, 2))
        out = C.c_uint64()
        if self.L.or_automorphism_count(k, _p(q, C.c_int32), len(q), C.byref(out)):
            raise OracleError(8, "automorphism search supports k <= 10")
        return out.value

    def normalization_factor(self, k) -> float:
        return self.L.or_normalization_factor(k)

    def cv(self, counts) -> float:
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        return self.L.or_coefficient_of_variation(_p(c, C.c_uint64), len(c))


class Reference:
    """The unmodified reference library (oracle/_ref/libmotif_ref.so)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(path)
        P = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        for name, args in {
            "ref_graph_new": [C.c_uint32, u32p, u32p, C.c_uint64, C.POINTER(P)],
            "ref_graph_csr": [P, u64p, u32p],
            "ref_graph_ranks": [P, u32p],
            "ref_random_coloring": [P, C.c_int, C.c_uint64, u8p],
            "ref_plan_new": [C.c_int, i32p, C.c_int, C.c_uint64, C.POINTER(P)],
            "ref_plan_canonical": [P, C.c_int, C.c_char_p, C.c_int],
            "ref_count_colorful": [P, u8p, C.c_int, P, C.c_int, C.c_int, C.c_int, u64p],
            "ref_count_ops": [P, u8p, C.c_int, P, C.c_int, u64p, u64p],
            "ref_count_batch": [P, u8p, C.c_int, C.c_int, P, C.c_int, C.c_int, C.c_int, u64p],
            "ref_brute_colorful": [P, P, u8p, C.c_int, C.c_uint64, u64p],
            "ref_brute_matches": [P, P, C.c_uint64, u64p],
            "ref_automorphism_count": [P, u64p],
            "ref_estimate": [P, P, C.c_int, C.c_uint64, C.c_uint64, u64p, C.POINTER(C.c_double),
                             C.POINTER(C.c_double), C.POINTER(C.c_double)],
        }.items():
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = args
        L.ref_graph_free.argtypes = [P]
        L.ref_graph_free.restype = None
        L.ref_plan_free.argtypes = [P]
        L.ref_plan_free.restype = None
        L.ref_graph_num_edges.argtypes = [P]
        L.ref_graph_num_edges.restype = C.c_uint64
        L.ref_plan_num_trees.argtypes = [P]
        L.ref_plan_num_trees.restype = C.c_int
        L.ref_normalization_factor.argtypes = [C.c_int]
        L.ref_normalization_factor.restype = C.c_double
        self.L = L

    def _ck(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    class Graph:
        def __init__(self, ref, n, edges):
            e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
            eu, ev = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
            self.ref, self.n = ref, n
            self.h = C.c_void_p()
            ref._ck(ref.L.ref_graph_new(n, _p(eu, C.c_uint32), _p(ev, C.c_uint32), len(e), C.byref(self.h)))
            self.m = ref.L.ref_graph_num_edges(self.h)

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.L.ref_graph_free(self.h)
                self.h = None

        def csr(self):
            off = np.empty(self.n + 1, dtype=np.uint64)
            adj = np.empty(max(2 * self.m, 1), dtype=np.uint32)
            self.ref._ck(self.ref.L.ref_graph_csr(self.h, _p(off, C.c_uint64), _p(adj, C.c_uint32)))
            return off, adj[: 2 * self.m]

        def ranks(self):
            r = np.empty(max(self.n, 1), dtype=np.uint32)
            self.ref._ck(self.ref.L.ref_graph_ranks(self.h, _p(r, C.c_uint32)))
            return r[: self.n]

        def coloring(self, k, seed):
            chi = np.empty(max(self.n, 1), dtype=np.uint8)
            self.ref._ck(self.ref.L.ref_random_coloring(self.h, k, seed, _p(chi, C.c_uint8)))
            return chi[: self.n]

    class Plan:
        def __init__(self, ref, k, qedges, max_trees=10000):
            q = np.ascontiguousarray(np.asarray(qedges, dtype=np.int32).reshape(-1, 2))
            self.ref, self.k = ref, k
            self.h = C.c_void_p()
            ref._ck(ref.L.ref_plan_new(k, _p(q, C.c_int32), len(q), max_trees, C.byref(self.h)))

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.L.ref_plan_free(self.h)
                self.h = None

        def num_trees(self):
            return self.ref.L.ref_plan_num_trees(self.h)

        def canonical(self, idx=-1):
            buf = C.create_string_buffer(1 << 16)
            self.ref._ck(self.ref.L.ref_plan_canonical(self.h, idx, buf, len(buf)))
            return buf.value.decode()

    def graph(self, n, edges):
        return Reference.Graph(self, n, edges)

    def plan(self, k, qedges, max_trees=10000):
        return Reference.Plan(self, k, qedges, max_trees)

    def count(self, g, plan, chi, engine=1, workers=1, tree=-1) -> int:
        out = C.c_uint64()
        c = np.ascontiguousarray(chi, dtype=np.uint8)
        self._ck(self.L.ref_count_colorful(g.h, _p(c, C.c_uint8), plan.k, plan.h, tree, engine, workers,
                                           C.byref(out)))
        return out.value

    def count_batch(self, g, plan, chis, engine=1, threads=1, workers=1):
        """threads colourings at a time; workers > 1 runs each through the
        reference's BSP executor (parallel_count) on that many OpenMP workers."""
        c = np.ascontiguousarray(chis, dtype=np.uint8)
        out = np.zeros(c.shape[0], dtype=np.uint64)
        self._ck(self.L.ref_count_batch(g.h, _p(c, C.c_uint8), c.shape[0], plan.k, plan.h, engine, threads,
                                        workers, _p(out, C.c_uint64)))
        return out

    def count_ops(self, g, plan, chi, engine=1):
        cnt, ops = C.c_uint64(), C.c_uint64()
        c = np.ascontiguousarray(chi, dtype=np.uint8)
        self._ck(self.L.ref_count_ops(g.h, _p(c, C.c_uint8), plan.k, plan.h, engine, C.byref(cnt), C.byref(ops)))
        return cnt.value, ops.value

    def brute_colorful(self, g, plan, chi, budget=10**9) -> int:
        out = C.c_uint64()
        c = np.ascontiguousarray(chi, dtype=np.uint8)
        self._ck(self.L.ref_brute_colorful(g.h, plan.h, _p(c, C.c_uint8), plan.k, budget, C.byref(out)))
        return out.value

    def brute_matches(self, g, plan, budget=10**9) -> int:
        out = C.c_uint64()
        self._ck(self.L.ref_brute_matches(g.h, plan.h, budget, C.byref(out)))
        return out.value

    def automorphism_count(self, plan) -> int:
        out = C.c_uint64()
        self._ck(self.L.ref_automorphism_count(plan.h, C.byref(out)))
        return out.value

    def estimate(self, g, plan, engine, trials, seed):
        per = np.zeros(trials, dtype=np.uint64)
        mean, cv, sub = C.c_double(), C.c_double(), C.c_double()
        self._ck(self.L.ref_estimate(g.h, plan.h, engine, trials, seed, _p(per, C.c_uint64), C.byref(mean),
                                     C.byref(cv), C.byref(sub)))
        return per, mean.value, cv.value, sub.value


def reference_available() -> bool:
    return os.path.exists(REF_LIB)
