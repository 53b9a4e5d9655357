"""B200-native direction-optimized BFS (arxiv 1503.04359 hot path) -- Python binding.

Argument marshalling only: every step of construction and traversal runs in
``libbfsb200.so``'s CUDA kernels behind the C ABI in ``include/bfs.h``.  The
functions below carry the C names; ``Graph`` is a small convenience wrapper
over them.  torch is used for device memory and streams only.

There is no CPU fallback: if the shared library is missing, importing the
binding raises; if no CUDA device is usable, the C calls fail with
``BFS_ERR_CUDA``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbfsb200.so")

BFS_OK = 0
STATUS_NAMES = {0: "BFS_OK", 1: "BFS_ERR_INVALID_ARG", 2: "BFS_ERR_OUT_OF_RANGE", 3: "BFS_ERR_MALFORMED_INPUT",
                4: "BFS_ERR_CAPACITY", 5: "BFS_ERR_OUT_OF_MEMORY", 6: "BFS_ERR_CUDA", 7: "BFS_ERR_NCCL",
                8: "BFS_ERR_INTERNAL"}
SRC_EDGES, SRC_CSR, SRC_KRONECKER = 0, 1, 2
KRON_ABC = (5700, 1900, 1900)
ER_ABC = (2500, 2500, 2500)

# exported symbols declared in include/bfs.h (checked by tests/test_abi.py)
EXPORTS = ("bfs_graph_create", "bfs_graph_create_kronecker", "bfs_graph_create_edges", "bfs_graph_create_csr",
           "bfs_graph_info", "bfs_graph_build_ms", "bfs_set_policy", "bfs_run", "bfs_stats", "bfs_graph_destroy",
           "bfs_comm_unique_id", "bfs_comm_create", "bfs_comm_create_local", "bfs_comm_destroy", "bfs_last_error",
           "bfs_kronecker_edges", "bfs_graph_export_csr", "bfs_graph_export_labels", "bfs_sample_roots",
           "bfs_set_allocator", "bfs_abi_version", "bfs_partition_range", "bfs_graph_export_row", "bfs_component_tuples",
           "bfs_validate", "bfs_graph_active", "bfs_graph_tiles")


class BfsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class bfs_kron_spec(ctypes.Structure):
    _fields_ = [("scale", ctypes.c_uint32), ("edgefactor", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("a", ctypes.c_uint32), ("b", ctypes.c_uint32), ("c", ctypes.c_uint32)]


class bfs_build_opts(ctypes.Structure):
    _fields_ = [("dedup", ctypes.c_int), ("drop_self_loops", ctypes.c_int), ("reindex_by_degree", ctypes.c_int),
                ("sort_rows", ctypes.c_int)]


class bfs_policy(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("alpha", ctypes.c_int64), ("beta", ctypes.c_int64),
                ("bu_from_level", ctypes.c_int), ("level_times", ctypes.c_int), ("loop", ctypes.c_int)]


class bfs_level_stats(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int), ("direction", ctypes.c_int), ("frontier", ctypes.c_int64),
                ("discovered", ctypes.c_int64), ("m_f", ctypes.c_int64), ("m_u", ctypes.c_int64),
                ("inspections", ctypes.c_int64), ("scanned", ctypes.c_int64), ("ms", ctypes.c_float),
                ("kernel_ms", ctypes.c_float), ("nvlink_bytes", ctypes.c_uint64)]


class bfs_run_stats(ctypes.Structure):
    _fields_ = [("root", ctypes.c_int64), ("reached", ctypes.c_int64), ("component_edge_tuples", ctypes.c_int64),
                ("levels", ctypes.c_int), ("ms_total", ctypes.c_double), ("ms_init", ctypes.c_double),
                ("ms_compute", ctypes.c_double), ("ms_push", ctypes.c_double), ("ms_pull", ctypes.c_double),
                ("ms_aggregate", ctypes.c_double), ("nvlink_bytes", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_int64)]


class bfs_graph_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("n", ctypes.c_int64), ("uv", ctypes.c_void_p), ("m", ctypes.c_int64),
                ("offsets", ctypes.c_void_p), ("adj", ctypes.c_void_p), ("kron", bfs_kron_spec),
                ("opts", bfs_build_opts)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libbfsb200.so (built by __graft_entry__.build() / build.py); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, i32, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int
        sig = {
            "bfs_graph_create": [P, P, P, P],
            "bfs_graph_create_kronecker": [P, P, P, P, P],
            "bfs_graph_create_edges": [P, i64, i64, P, P, P, P],
            "bfs_graph_create_csr": [P, P, i64, P, P, P, P],
            "bfs_graph_info": [P, P, P, P, P],
            "bfs_graph_build_ms": [P, P],
            "bfs_set_policy": [P, P],
            "bfs_run": [P, i64, P, P],
            "bfs_stats": [P, P, P, i32],
            "bfs_graph_destroy": [P],
            "bfs_comm_unique_id": [P],
            "bfs_comm_create": [i32, i32, P, i32, P],
            "bfs_comm_create_local": [i32, i32, P],
            "bfs_comm_destroy": [P],
            "bfs_kronecker_edges": [P, i64, i64, P, P],
            "bfs_graph_export_csr": [P, P, P],
            "bfs_graph_export_labels": [P, P],
            "bfs_sample_roots": [P, ctypes.c_uint32, ctypes.c_uint64, i64, P, P],
            "bfs_set_allocator": [P, P, P],
            "bfs_partition_range": [i64, i32, i32, P, P],
            "bfs_graph_export_row": [P, i64, P, i64, P],
            "bfs_component_tuples": [P, P],
            "bfs_validate": [P, i64, P, P, P],
            "bfs_graph_active": [P, P],
            "bfs_graph_tiles": [P, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = st
        L.bfs_last_error.argtypes = []
        L.bfs_last_error.restype = ctypes.c_char_p
        L.bfs_abi_version.argtypes = []
        L.bfs_abi_version.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != BFS_OK:
        raise BfsError(status, lib().bfs_last_error().decode(errors="replace"))


def _ptr(x) -> int | None:
    """Raw address of a torch tensor / numpy array (or None)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    return int(x)


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


def default_opts(dedup=True, drop_self_loops=True, reindex_by_degree=False, sort_rows=1) -> bfs_build_opts:
    """sort_rows: 0 fill order, 1 ascending neighbour ID, 2 decreasing neighbour degree."""
    return bfs_build_opts(int(dedup), int(drop_self_loops), int(reindex_by_degree), int(sort_rows))


# ----------------------------------------------------------------------------- C-named wrappers
def bfs_graph_create_kronecker(scale: int, edgefactor: int = 16, seed: int = 1, abc=KRON_ABC, opts=None, comm=None,
                               stream=None) -> ctypes.c_void_p:
    spec = bfs_kron_spec(scale, edgefactor, seed, *abc)
    h = ctypes.c_void_p()
    o = opts or default_opts()
    _check(lib().bfs_graph_create_kronecker(ctypes.byref(spec), ctypes.byref(o), comm, _stream_ptr(stream),
                                            ctypes.byref(h)))
    return h


def bfs_graph_create_edges(uv, n: int, opts=None, comm=None, stream=None) -> ctypes.c_void_p:
    m = int(uv.shape[0]) if uv is not None else 0
    h = ctypes.c_void_p()
    o = opts or default_opts()
    _check(lib().bfs_graph_create_edges(_ptr(uv) if m else None, m, n, ctypes.byref(o), comm, _stream_ptr(stream),
                                        ctypes.byref(h)))
    return h


def bfs_graph_create_csr(offsets, adj, n: int, opts=None, comm=None, stream=None) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    o = opts or default_opts()
    _check(lib().bfs_graph_create_csr(_ptr(offsets), _ptr(adj), n, ctypes.byref(o), comm, _stream_ptr(stream),
                                      ctypes.byref(h)))
    return h


def bfs_graph_info(h):
    v = [ctypes.c_int64() for _ in range(4)]
    _check(lib().bfs_graph_info(h, *[ctypes.byref(x) for x in v]))
    return tuple(x.value for x in v)


def bfs_graph_active(h) -> int:
    """Vertices the per-search bitmaps cover (non-isolated prefix when reindexed on one GPU)."""
    x = ctypes.c_int64()
    _check(lib().bfs_graph_active(h, ctypes.byref(x)))
    return x.value


def bfs_graph_tiles(h) -> dict:
    """Tiled top-down index: heavy rows, label tiles (0 = none), index build ms."""
    hr, t, ms = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    _check(lib().bfs_graph_tiles(h, ctypes.byref(hr), ctypes.byref(t), ctypes.byref(ms)))
    return {"heavy_rows": hr.value, "tiles": t.value, "build_ms": ms.value}


def bfs_graph_build_ms(h) -> float:
    x = ctypes.c_double()
    _check(lib().bfs_graph_build_ms(h, ctypes.byref(x)))
    return x.value


LOOPS = {"auto": 0, "host": 1, "graph": 2, "persistent": 3, "cluster": 4}


def bfs_set_policy(h, mode: int = 0, alpha: int = 15, beta: int = 18, bu_from_level: int = 0, level_times: bool = False,
                   loop="auto", host_loop: bool = False):
    """loop: 'auto' | 'host' | 'graph' | 'persistent' | 'cluster' (or 0..4); host_loop=True is loop='host'."""
    lp = 1 if host_loop else (LOOPS[loop] if isinstance(loop, str) else int(loop))
    p = bfs_policy(mode, alpha, beta, bu_from_level, int(level_times), lp)
    _check(lib().bfs_set_policy(h, ctypes.byref(p)))


def _check_output(x, nl: int, name: str):
    """An output buffer must be int32, contiguous and hold the nl owned vertices, in
    device memory of the current device or in (pinned or pageable) host memory."""
    if x is None:
        return
    if hasattr(x, "data_ptr"):       # torch tensor
        import torch
        if x.dtype != torch.int32:
            raise ValueError(f"{name}: dtype {x.dtype}, expected torch.int32")
        if not x.is_contiguous():
            raise ValueError(f"{name}: not contiguous")
        if x.numel() < nl:
            raise ValueError(f"{name}: {x.numel()} elements < {nl} owned vertices")
        if x.is_cuda and x.device.index != torch.cuda.current_device():
            raise ValueError(f"{name}: on {x.device}, the graph's device is cuda:{torch.cuda.current_device()}")
    elif isinstance(x, np.ndarray):
        if x.dtype != np.int32 or not x.flags["C_CONTIGUOUS"] or x.size < nl:
            raise ValueError(f"{name}: needs a contiguous int32 array of >= {nl} elements")
    else:
        raise ValueError(f"{name}: expected a torch tensor or numpy array, got {type(x).__name__}")


def bfs_run(h, root: int, parent_out, depth_out, check: bool = True):
    """parent_out / depth_out: int32 buffers of local_end - local_begin entries (device or host).
    check=False skips the buffer checks (timed loops that checked the same buffers once)."""
    if check:
        _, _, lo, hi = bfs_graph_info(h)
        _check_output(parent_out, hi - lo, "parent_out")
        _check_output(depth_out, hi - lo, "depth_out")
    _check(lib().bfs_run(h, int(root), _ptr(parent_out), _ptr(depth_out)))


def bfs_component_tuples(h) -> int:
    t = ctypes.c_int64()
    _check(lib().bfs_component_tuples(h, ctypes.byref(t)))
    return t.value


def bfs_stats(h, max_levels: int | None = None):
    """(run, levels) of the last search; every step record unless max_levels caps it."""
    rs = bfs_run_stats()
    if max_levels is None:
        _check(lib().bfs_stats(h, ctypes.byref(rs), None, 0))
        max_levels = max(1, rs.levels)
    lv = (bfs_level_stats * max_levels)()
    _check(lib().bfs_stats(h, ctypes.byref(rs), lv, max_levels))
    levels = [{f: getattr(lv[i], f) for f, _ in bfs_level_stats._fields_} for i in range(min(rs.levels, max_levels))]
    run = {f: getattr(rs, f) for f, _ in bfs_run_stats._fields_}
    return run, levels


VALIDATE_RULES = ("V1_root", "V2_tree_edge", "V3_parent_depth", "V4_edge_span", "V5_unreached")


def bfs_validate(h, root: int, parent, depth) -> dict:
    """Graph500 validation of one search's outputs on the device;
    {rule: violations} for failing rules only ({} = valid)."""
    f = np.zeros(5, np.int64)
    _check(lib().bfs_validate(h, int(root), _ptr(parent), _ptr(depth), _ptr(f)))
    return {VALIDATE_RULES[i]: int(f[i]) for i in range(5) if f[i]}


def bfs_graph_destroy(h):
    if h:
        _check(lib().bfs_graph_destroy(h))


def bfs_kronecker_edges(scale: int, edgefactor: int, seed: int, abc, first: int, count: int, uv_out, stream=None):
    spec = bfs_kron_spec(scale, edgefactor, seed, *abc)
    _check(lib().bfs_kronecker_edges(ctypes.byref(spec), first, count, _ptr(uv_out), _stream_ptr(stream)))


def bfs_graph_export_csr(h, offsets_out, adj_out):
    _check(lib().bfs_graph_export_csr(h, _ptr(offsets_out), _ptr(adj_out)))


def bfs_graph_export_row(h, v: int, cap: int = 1 << 20) -> np.ndarray:
    """Local row v (stored order), at most cap neighbours, as a host int32 array."""
    deg = ctypes.c_int64()
    _check(lib().bfs_graph_export_row(h, v, None, 0, ctypes.byref(deg)))
    out = np.empty(max(1, min(cap, deg.value)), np.int32)
    _check(lib().bfs_graph_export_row(h, v, _ptr(out), min(cap, deg.value), ctypes.byref(deg)))
    return out[: min(cap, deg.value)]


def bfs_graph_export_labels(h, out):
    _check(lib().bfs_graph_export_labels(h, _ptr(out)))


def bfs_sample_roots(h, scale: int, seed: int, count: int) -> np.ndarray:
    roots = np.zeros(max(count, 1), np.int64)
    found = ctypes.c_int64()
    _check(lib().bfs_sample_roots(h, scale, seed, count, _ptr(roots), ctypes.byref(found)))
    return roots[: found.value]


def bfs_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().bfs_comm_unique_id(buf))
    return bytes(buf)


def bfs_comm_create(nranks: int, rank: int, uid: bytes, device: int) -> ctypes.c_void_p:
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    _check(lib().bfs_comm_create(nranks, rank, buf, device, ctypes.byref(h)))
    return h


def bfs_comm_create_local(nparts: int, device: int = 0) -> list:
    """nparts rank endpoints in this process (one device); drive each from its own thread."""
    arr = (ctypes.c_void_p * nparts)()
    _check(lib().bfs_comm_create_local(nparts, device, arr))
    return [ctypes.c_void_p(arr[i]) for i in range(nparts)]


def bfs_partition_range(n: int, nranks: int, rank: int):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().bfs_partition_range(n, nranks, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def run_ranks(fn, nranks: int):
    """Call fn(rank) on nranks host threads (for local-comm partitions); re-raise the
    first failure.  ctypes releases the GIL inside library calls, so the ranks
    progress concurrently through their collectives."""
    import threading
    out = [None] * nranks
    err = []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


def bfs_comm_destroy(h):
    if h:
        _check(lib().bfs_comm_destroy(h))


# ----------------------------------------------------------------------------- convenience
class Graph:
    """Owns a bfs_graph_t.  Outputs are torch int32 tensors on the graph's device."""

    def __init__(self, handle, device=None, stream=None):
        import torch
        self.h = handle
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.stream = stream
        self.n, self.arcs, self.local_begin, self.local_end = bfs_graph_info(handle)

    @classmethod
    def kronecker(cls, scale, edgefactor=16, seed=1, abc=KRON_ABC, opts=None, comm=None, stream=None):
        return cls(bfs_graph_create_kronecker(scale, edgefactor, seed, abc, opts, comm, stream), stream=stream)

    @classmethod
    def from_edges(cls, uv, n, opts=None, comm=None, stream=None):
        return cls(bfs_graph_create_edges(uv, n, opts, comm, stream), stream=stream)

    @classmethod
    def from_csr(cls, offsets, adj, n, opts=None, comm=None, stream=None):
        return cls(bfs_graph_create_csr(offsets, adj, n, opts, comm, stream), stream=stream)

    @property
    def build_ms(self) -> float:
        return bfs_graph_build_ms(self.h)

    def set_policy(self, **kw):
        bfs_set_policy(self.h, **kw)

    def run(self, root: int, parent=None, depth=None):
        import torch
        nl = self.local_end - self.local_begin
        if parent is None:
            parent = torch.empty(nl, dtype=torch.int32, device=self.device)
        if depth is None:
            depth = torch.empty(nl, dtype=torch.int32, device=self.device)
        bfs_run(self.h, root, parent, depth)
        return parent, depth

    def stats(self, tuples: bool = True):
        """(run, levels) of the last run; tuples=True also reduces the TEPS numerator
        on the device (collective on p ranks; keep it out of timed loops)."""
        if tuples:
            bfs_component_tuples(self.h)
        return bfs_stats(self.h)

    def export_csr(self):
        import torch
        nl = self.local_end - self.local_begin
        off = torch.empty(nl + 1, dtype=torch.int64, device=self.device)
        bfs_graph_export_csr(self.h, off, None)
        adj = torch.empty(max(int(off[-1].item()), 1), dtype=torch.int32, device=self.device)
        bfs_graph_export_csr(self.h, None, adj)
        return off, adj[: int(off[-1].item())]

    def sample_roots(self, scale, seed, count=64):
        return bfs_sample_roots(self.h, scale, seed, count)

    def close(self):
        if self.h:
            bfs_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
