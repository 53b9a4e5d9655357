"""Parity oracle -- TEST INFRASTRUCTURE ONLY.

Plain serial CPU implementation (``oracle/oracle.c``, plain C, integer only) of
what the direction-optimized BFS hot path computes, plus thin numpy/ctypes
wrappers.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package; the product
package ``paper_1503_04359_b200`` never does, and shares no code with it.

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n.

Functions and the passage each follows:

* ``philox4x32_10``           -- counter-based RNG (R12)
* ``kron_edges``              -- Graph500 Kronecker generator
* ``build_csr``               -- CSR, each undirected edge as two arcs
* ``degree_reindex`` / ``relabel_csr`` -- section 3.4 locality reindex
* ``degree_reindex_local``   -- the same per partition: block partition, then local IDs
* ``sort_rows_by_degree``     -- section 3.4 row order without relabeling
* ``bfs``                     -- serial FIFO BFS, the plain definition
* ``validate``                -- Graph500 validator V1-V6
* ``stream_validate_edges`` / ``stream_validate_vertices`` -- the same rules V1-V5 over the
  input tuples of R searches at once
* ``do_emulate``              -- direction rule, counters, inspections
* ``component_tuples``, ``compute_teps``, ``harmonic_mean`` -- TEPS
* ``sample_roots``            -- seeded root list (R8)

Parity status: every function above is pinned by ``tests/test_oracle_*.py``
against values fixed independently of this code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

KRON_ABC = (5700, 1900, 1900)  # Graph500 A, B, C per 10000
ER_ABC = (2500, 2500, 2500)    # all quadrants equal: uniform random multigraph


def build_library(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O3 for an x86-64-v3 (AVX2) host: integer code only, so the flags
    cannot change a result; no OpenMP, no threads -- the harness runs ranges in parallel)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_library())
            i64, i32, u64, u32 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32
            P = ctypes.c_void_p
            lib.orc_philox4x32_10.argtypes = [P, P, P]
            lib.orc_kron_scramble_keys.argtypes = [u64, P]
            lib.orc_kron_scramble.argtypes = [i32, P, u32]
            lib.orc_kron_scramble.restype = u32
            lib.orc_kron_edges.argtypes = [i32, u64, u32, u32, u32, i64, i64, i32, P]
            lib.orc_build_csr.argtypes = [i64, i64, P, i32, i32, i32, P, P, P]
            lib.orc_build_csr.restype = i64
            lib.orc_degree_reindex.argtypes = [i64, P, i64, P, P]
            lib.orc_degree_reindex.restype = i32
            lib.orc_degree_reindex_local.argtypes = [i64, P, i64, P, P]
            lib.orc_degree_reindex_local.restype = i32
            lib.orc_relabel_csr.argtypes = [i64, P, P, P, P, P, P]
            lib.orc_sort_rows_by_degree.argtypes = [i64, P, P]
            lib.orc_bfs.argtypes = [i64, P, P, i64, P, P]
            lib.orc_bfs.restype = i64
            lib.orc_validate.argtypes = [i64, P, P, i64, P, P, P, P, P]
            lib.orc_validate.restype = i64
            lib.orc_stream_validate_edges.argtypes = [i64, i32, P, i64, i64, P, P, P, P, P]
            lib.orc_stream_validate_edges.restype = None
            lib.orc_stream_validate_vertices.argtypes = [i64, i32, P, P, P, P, i64, i64, P, P]
            lib.orc_stream_validate_vertices.restype = None
            lib.orc_do_emulate.argtypes = [i64, P, P, P, i64, i64, i32, i64, i64, P, P, P, P, P, P, P, i64]
            lib.orc_do_emulate.restype = i64
            lib.orc_component_tuples.argtypes = [i64, P, P]
            lib.orc_component_tuples.restype = i64
            lib.orc_sample_roots.argtypes = [i32, u64, i64, P, P, i64, i64, P]
            lib.orc_sample_roots.restype = i64
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------- RNG / generator
def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 of a 4-word counter under a 2-word key (Random123 definition)."""
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    _L().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def scramble_keys(seed: int) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    _L().orc_kron_scramble_keys(ctypes.c_uint64(seed), _p(out))
    return out


def scramble(scale: int, keys, v: int) -> int:
    k = _c(keys, np.uint32)
    return int(_L().orc_kron_scramble(scale, _p(k), v))


def kron_edges(scale: int, edgefactor: int = 16, seed: int = 1, abc=KRON_ABC, first: int = 0,
               count: int | None = None, scramble_labels: bool = True) -> np.ndarray:
    """Edge tuples [first, first+count) of the Kronecker graph, int32 [count, 2]."""
    m = edgefactor << scale
    if count is None:
        count = m - first
    uv = np.zeros((count, 2), np.int32)
    a, b, c = abc
    _L().orc_kron_edges(scale, ctypes.c_uint64(seed), a, b, c, first, count, 1 if scramble_labels else 0, _p(uv))
    return uv


# --------------------------------------------------------------------------- CSR
class CSR:
    """offsets int64[n+1], adj int32[arcs]."""

    def __init__(self, n: int, offsets: np.ndarray, adj: np.ndarray):
        self.n = int(n)
        self.offsets = offsets
        self.adj = adj

    @property
    def arcs(self) -> int:
        return int(self.offsets[-1])

    def degree(self, v: int | None = None):
        d = np.diff(self.offsets)
        return d if v is None else int(d[v])

    def row(self, v: int) -> np.ndarray:
        return self.adj[self.offsets[v]:self.offsets[v + 1]]


class MalformedInput(ValueError):
    pass


def build_csr(n: int, uv, dedup: bool = False, drop_self_loops: bool = False, sort_rows: bool = False) -> CSR:
    """S:44-52 build_csr; raises MalformedInput naming the bad tuple."""
    uv = _c(np.asarray(uv).reshape(-1, 2) if len(uv) else np.zeros((0, 2)), np.int32)
    m = uv.shape[0]
    offsets = np.zeros(n + 1, np.int64)
    adj = np.zeros(max(2 * m, 1), np.int32)
    arcs = np.zeros(1, np.int64)
    rc = _L().orc_build_csr(n, m, _p(uv), int(dedup), int(drop_self_loops), int(sort_rows),
                            _p(offsets), _p(adj), _p(arcs))
    if rc < 0:
        k = -rc - 1
        raise MalformedInput(f"tuple {k} = ({uv[k, 0]}, {uv[k, 1]}) has an endpoint outside [0, {n})")
    return CSR(n, offsets, adj[: int(arcs[0])].copy())


def degree_reindex(g: CSR, p: int = 1):
    """(new_label int64[n], position int64[n]) by (degree desc, ID asc), dealt round-robin to p parts."""
    new_label = np.zeros(g.n, np.int64)
    position = np.zeros(g.n, np.int64)
    rc = _L().orc_degree_reindex(g.n, _p(g.offsets), p, _p(new_label), _p(position))
    if rc != 0:
        raise ValueError("p must divide n")
    return new_label, position


def degree_reindex_local(g: CSR, p: int = 1):
    """(new_label int64[n], position int64[n]): the 1D block partition first (p blocks of
    n/p original labels), then each block numbers its own vertices by (degree desc, ID asc)
    ("permutation of local IDs"); position = global (degree desc, ID asc) place."""
    new_label = np.zeros(g.n, np.int64)
    position = np.zeros(g.n, np.int64)
    rc = _L().orc_degree_reindex_local(g.n, _p(g.offsets), p, _p(new_label), _p(position))
    if rc != 0:
        raise ValueError("p must divide n")
    return new_label, position


def relabel_csr(g: CSR, new_label: np.ndarray, position: np.ndarray) -> CSR:
    offsets = np.zeros(g.n + 1, np.int64)
    adj = np.zeros(max(g.arcs, 1), np.int32)
    nl = _c(new_label, np.int64)
    pos = _c(position, np.int64)
    _L().orc_relabel_csr(g.n, _p(g.offsets), _p(g.adj), _p(nl), _p(pos), _p(offsets), _p(adj))
    return CSR(g.n, offsets, adj[: g.arcs].copy())


def sort_rows_by_degree(g: CSR) -> CSR:
    """Rows by decreasing neighbour degree, ties by ascending ID; labels unchanged."""
    adj = g.adj.copy()
    if g.arcs:
        _L().orc_sort_rows_by_degree(g.n, _p(g.offsets), _p(adj))
    return CSR(g.n, g.offsets.copy(), adj)


# --------------------------------------------------------------------------- BFS / validation
def bfs(g: CSR, root: int):
    """Serial FIFO BFS -> (depth int32[n], parent int32[n]); -1 = unreached."""
    if not (0 <= root < g.n):
        raise IndexError(f"root {root} outside [0, {g.n})")
    depth = np.empty(g.n, np.int32)
    parent = np.empty(g.n, np.int32)
    _L().orc_bfs(g.n, _p(g.offsets), _p(g.adj if g.arcs else np.zeros(1, np.int32)), root, _p(depth), _p(parent))
    return depth, parent


RULES = ("V1_root", "V2_tree_edge", "V3_parent_depth", "V4_edge_span", "V5_unreached", "V6_exact_depth")


def validate(g: CSR, root: int, depth, parent, ref_depth=None) -> dict:
    """Graph500 validator; returns {rule: (fail_count, first_bad_vertex)} for failing rules only."""
    d = _c(depth, np.int32)
    p = _c(parent, np.int32)
    r = _c(ref_depth, np.int32) if ref_depth is not None else None
    fails = np.zeros(6, np.int64)
    first = np.zeros(6, np.int64)
    adj = g.adj if g.arcs else np.zeros(1, np.int32)
    _L().orc_validate(g.n, _p(g.offsets), _p(adj), root, _p(d), _p(p), _p(r) if r is not None else None,
                      _p(fails), _p(first))
    return {RULES[i]: (int(fails[i]), int(first[i])) for i in range(6) if fails[i]}


STREAM_RULES = ("V1_root", "V2_tree_edge", "V3_parent_depth", "V4_edge_span", "V5_unreached")


def stream_validate_edges(n: int, uv, index0: int, depth8, parent, witness):
    """Edge pass of the streaming validator over tuples uv (int32 [k, 2], tuple indices
    index0..index0+k); depth8 int8 [n, R], parent int32 [n, R], witness uint8 [n, R]
    (updated).  Returns (fails_v4 int64[R], first_v4 int64[R]).  Releases the GIL
    (ctypes), so disjoint tuple ranges can be checked from several threads."""
    R = depth8.shape[1]
    assert depth8.dtype == np.int8 and parent.dtype == np.int32 and witness.dtype == np.uint8
    assert depth8.shape == parent.shape == witness.shape == (n, R)
    assert depth8.flags["C_CONTIGUOUS"] and parent.flags["C_CONTIGUOUS"] and witness.flags["C_CONTIGUOUS"]
    uv = _c(uv, np.int32)
    fails = np.zeros(R, np.int64)
    first = np.full(R, -1, np.int64)
    _L().orc_stream_validate_edges(n, R, _p(uv), uv.shape[0], index0, _p(depth8), _p(parent), _p(witness),
                                   _p(fails), _p(first))
    return fails, first


def stream_validate_vertices(n: int, roots, depth8, parent, witness, v0: int = 0, v1: int | None = None):
    """Vertex pass (V1, V2, V3, V5) over [v0, v1) after the edge pass saw every tuple.
    Returns (fails int64[R, 5], first int64[R, 5]); column 3 (V4) stays 0."""
    R = depth8.shape[1]
    v1 = n if v1 is None else v1
    rt = _c(roots, np.int64)
    assert rt.shape == (R,)
    fails = np.zeros((R, 5), np.int64)
    first = np.full((R, 5), -1, np.int64)
    _L().orc_stream_validate_vertices(n, R, _p(rt), _p(depth8), _p(parent), _p(witness), v0, v1, _p(fails),
                                      _p(first))
    return fails, first


def do_emulate(g: CSR, depth, alpha: int = 15, beta: int = 18, policy: int = 0, bu_from: int = 0,
               want_bu_parent: bool = False, coord_hi: int | None = None) -> dict:
    """Per-step direction, n_f, m_f, m_u, discovered and inspections (see oracle.c).
    coord_hi: policy 3's coordinator owns labels [0, coord_hi) (default: all)."""
    d = _c(depth, np.int32)
    S = int(d.max()) + 2 if d.size else 2
    dirs = np.zeros(S, np.int32)
    arrs = [np.zeros(S, np.int64) for _ in range(5)]
    bp = np.zeros(g.n, np.int32) if want_bu_parent else None
    adj = g.adj if g.arcs else np.zeros(1, np.int32)
    steps = _L().orc_do_emulate(g.n, _p(g.offsets), _p(adj), _p(d), alpha, beta, policy, bu_from, S,
                                _p(dirs), *[_p(a) for a in arrs], _p(bp) if bp is not None else None,
                                g.n if coord_hi is None else int(coord_hi))
    assert steps >= 0
    out = {"dir": dirs[:steps], "n_f": arrs[0][:steps], "m_f": arrs[1][:steps], "m_u": arrs[2][:steps],
           "discovered": arrs[3][:steps], "insp": arrs[4][:steps]}
    if bp is not None:
        out["bu_parent"] = bp
    return out


# --------------------------------------------------------------------------- TEPS
def component_tuples(uv, depth) -> int:
    uv = _c(np.asarray(uv).reshape(-1, 2), np.int32)
    d = _c(depth, np.int32)
    return int(_L().orc_component_tuples(uv.shape[0], _p(uv), _p(d)))


def compute_teps(edges: int, seconds: float) -> float:
    """edges / elapsed; elapsed must be > 0."""
    if not seconds > 0:
        raise ValueError("elapsed must be > 0")
    return edges / seconds


def harmonic_mean(rates) -> float:
    """n / sum(1/rate); rates must be non-empty and positive."""
    rates = list(rates)
    if not rates or any(not r > 0 for r in rates):
        raise ValueError("harmonic mean needs a non-empty list of positive rates")
    return len(rates) / sum(1.0 / r for r in rates)


def sample_roots(g: CSR, scale: int, seed: int, count: int = 64, max_candidates: int | None = None) -> np.ndarray:
    if max_candidates is None:
        max_candidates = max(64 * count, 4 * g.n)
    roots = np.zeros(count, np.int64)
    adj = g.adj if g.arcs else np.zeros(1, np.int32)
    got = _L().orc_sample_roots(scale, ctypes.c_uint64(seed), g.n, _p(g.offsets), _p(adj), count,
                                max_candidates, _p(roots))
    return roots[:got]


def kron_graph(scale: int, edgefactor: int = 16, seed: int = 1, abc=KRON_ABC, dedup: bool = True,
               drop_self_loops: bool = True, sort_rows: bool = True):
    """Convenience: (uv, CSR) of a generated graph, built entirely by the oracle."""
    uv = kron_edges(scale, edgefactor, seed, abc)
    return uv, build_csr(1 << scale, uv, dedup=dedup, drop_self_loops=drop_self_loops, sort_rows=sort_rows)
