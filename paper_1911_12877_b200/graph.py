"""Host-side graph object and the device-resident replica cache.

Mirrors the reference's ``Graph`` (proj/include/symmine/graph.hpp:20-59,
python/module.cpp:111-139): an immutable CSR with strictly ascending,
symmetric neighbour lists, no self loops, ``size_t`` offsets and ``uint32``
ids.  ``Graph.from_edges`` builds exactly the layout of ``Graph::from_edges``
(graph.cpp:13-47) in native code (libsymmine_graph.so).  The device copy is
uploaded once per device set and cached on the object, matching the
reference's contract that a Graph is immutable after construction
(graph.hpp:18-19).
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N


def _csr_take(handle) -> tuple[np.ndarray, np.ndarray, int]:
    lib = N.graph_lib()
    n, s, m = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    N.check_graph(lib.smg_csr_info(handle, ctypes.byref(n), ctypes.byref(s), ctypes.byref(m)))
    off = np.ctypeslib.as_array(lib.smg_csr_offsets(handle), shape=(n.value + 1,)).copy()
    if s.value:
        adj = np.ctypeslib.as_array(lib.smg_csr_adjacency(handle), shape=(s.value,)).copy()
    else:
        adj = np.zeros(0, dtype=np.uint32)
    lib.smg_csr_free(handle)
    return off, adj, m.value


class Graph:
    """Sorted symmetric CSR graph (uint32 ids, uint64 offsets)."""

    def __init__(self, offsets, adjacency, *, max_degree: int | None = None, check: bool = True,
                 stats: tuple[int, int] = (0, 0)):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.adjacency = np.ascontiguousarray(adjacency, dtype=np.uint32)
        if self.offsets.ndim != 1 or self.offsets.size < 1:
            raise N.InputError("offsets must be a 1-D array of length n+1")
        if check:
            _check_csr(self.offsets, self.adjacency)
        deg = np.diff(self.offsets)
        self._max_degree = int(deg.max()) if deg.size else 0
        self.duplicate_edges, self.self_loops = stats
        self._dev = {}
        self._dev_lock = threading.Lock()

    # --- construction ----------------------------------------------------
    @staticmethod
    def from_edges(n: int, edges) -> "Graph":
        """Graph::from_edges (graph.cpp:13-47): symmetrise, drop self loops and
        duplicates (counted in .duplicate_edges / .self_loops)."""
        pairs = np.ascontiguousarray(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
        if pairs.size and (pairs.min() < 0 or pairs.max() >= n):
            raise N.InputError("edge endpoint out of range")
        pairs = pairs.astype(np.uint32)
        lib = N.graph_lib()
        h = ctypes.c_void_p()
        d, s = ctypes.c_uint64(), ctypes.c_uint64()
        ptr = pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if pairs.size else None
        N.check_graph(lib.smg_csr_from_edges(n, ptr, pairs.shape[0], ctypes.byref(h), ctypes.byref(d),
                                             ctypes.byref(s)))
        off, adj, m = _csr_take(h)
        return Graph(off, adj, max_degree=m, check=False, stats=(d.value, s.value))

    @staticmethod
    def from_csr(offsets, adjacency) -> "Graph":
        return Graph(offsets, adjacency)

    @staticmethod
    def _from_handle(h) -> "Graph":
        off, adj, m = _csr_take(h)
        return Graph(off, adj, max_degree=m, check=False)

    # --- accessors (graph.hpp:34-41) ---------------------------------------
    @property
    def n(self) -> int:
        return int(self.offsets.size - 1)

    @property
    def m(self) -> int:
        return int(self.adjacency.size // 2)

    @property
    def max_degree(self) -> int:
        return self._max_degree

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def neighbors(self, v: int) -> list[int]:
        return self.adjacency[int(self.offsets[v]):int(self.offsets[v + 1])].tolist()

    def orient(self) -> "Graph":
        """orient_reindex (graph.cpp:137-161): ids by (degree desc, id asc)."""
        return self.orient_with_map()[0]

    def orient_with_map(self):
        lib = N.graph_lib()
        src = _to_handle(self)
        try:
            h = ctypes.c_void_p()
            n2o = np.zeros(max(self.n, 1), dtype=np.uint32)
            N.check_graph(lib.smg_csr_orient(src, ctypes.byref(h),
                                             n2o.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
        finally:
            lib.smg_csr_free(src)
        return Graph._from_handle(h), n2o[: self.n]

    def __eq__(self, other) -> bool:  # graph.hpp:50-52
        return (isinstance(other, Graph) and np.array_equal(self.offsets, other.offsets)
                and np.array_equal(self.adjacency, other.adjacency))

    def __repr__(self) -> str:
        return f"Graph(n={self.n}, m={self.m})"

    # --- device replicas ---------------------------------------------------
    def device_handle(self, devices: tuple[int, ...]):
        """smg_graph* replicated on `devices` (uploaded once, then cached)."""
        with self._dev_lock:
            h = self._dev.get(devices)
            if h is None:
                lib = N.gpu_lib()
                out = ctypes.c_void_p()
                dev_arr = (ctypes.c_int * len(devices))(*devices)
                adj = self.adjacency if self.adjacency.size else np.zeros(1, dtype=np.uint32)
                N.check_gpu(lib.smg_graph_create(
                    self.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                    adj.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), self.n, dev_arr,
                    len(devices), ctypes.byref(out)))
                h = out
                self._dev[devices] = h
            return h

    def release_device(self) -> None:
        with self._dev_lock:
            if self._dev:
                lib = N.gpu_lib()
                for h in self._dev.values():
                    lib.smg_graph_destroy(h)
                self._dev.clear()

    def __del__(self):
        try:
            self.release_device()
        except Exception:
            pass


def _adopt_device(h, device: int) -> Graph:
    """Download a device-built graph handle and keep it as the Graph's replica."""
    lib = N.gpu_lib()
    n, s, m, nd = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int()
    N.check_gpu(lib.smg_graph_info(h, ctypes.byref(n), ctypes.byref(s), ctypes.byref(m),
                                   ctypes.byref(nd)))
    off = np.zeros(n.value + 1, dtype=np.uint64)
    adj = np.zeros(max(s.value, 1), dtype=np.uint32)
    N.check_gpu(lib.smg_graph_download(h, 0, off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                       adj.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    g = Graph(off, adj[: s.value], check=False)
    g._dev[(device,)] = h
    return g


def from_edges_device(n: int, edges, device: int = 0) -> Graph:
    """Graph::from_edges (graph.cpp:13-47) built on the GPU (radix sorts);
    structurally equal to Graph.from_edges.  The device copy is kept."""
    pairs = np.ascontiguousarray(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    if pairs.size and (pairs.min() < 0 or pairs.max() >= n):
        raise N.InputError("edge endpoint out of range")
    pairs = pairs.astype(np.uint32)
    lib = N.gpu_lib()
    h = ctypes.c_void_p()
    d, s = ctypes.c_uint64(), ctypes.c_uint64()
    dev = (ctypes.c_int * 1)(device)
    ptr = pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if pairs.size else None
    N.check_gpu(lib.smg_graph_from_edges(ptr, pairs.shape[0], n, dev, 1, ctypes.byref(h),
                                         ctypes.byref(d), ctypes.byref(s)))
    g = _adopt_device(h, device)
    g.duplicate_edges, g.self_loops = d.value, s.value
    return g


def orient_device(g: Graph, device: int = 0):
    """orient_reindex (graph.cpp:137-161) on the GPU -> (Graph, new_to_old)."""
    lib = N.gpu_lib()
    src = g.device_handle((device,))
    h = ctypes.c_void_p()
    n2o = np.zeros(max(g.n, 1), dtype=np.uint32)
    N.check_gpu(lib.smg_graph_orient(src, 0, ctypes.byref(h),
                                     n2o.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    return _adopt_device(h, device), n2o[: g.n]


def _check_csr(off: np.ndarray, adj: np.ndarray) -> None:
    n = off.size - 1
    if int(off[0]) != 0 or int(off[-1]) != adj.size:
        raise N.InputError("offsets must start at 0 and end at len(adjacency)")
    deg = np.diff(off.astype(np.int64))
    if (deg < 0).any():
        raise N.InputError("offsets must be non-decreasing")
    if adj.size:
        if int(adj.max()) >= n:
            raise N.InputError("adjacency id out of range")
        src = np.repeat(np.arange(n, dtype=np.int64), deg)
        if (adj.astype(np.int64) == src).any():
            raise N.InputError("self loop in adjacency")
        same = src[1:] == src[:-1]
        if (adj[1:][same] <= adj[:-1][same]).any():
            raise N.InputError("neighbour lists must be strictly ascending")
        # symmetry (graph.hpp:18-19): every slot (v, x) has its reverse (x, v);
        # rows ascending + lists ascending -> the keys are already sorted
        keys = src * n + adj.astype(np.int64)
        rev = adj.astype(np.int64) * n + src
        pos = np.minimum(np.searchsorted(keys, rev), keys.size - 1)
        if (keys[pos] != rev).any():
            raise N.InputError("adjacency must be symmetric (missing reverse edge)")


def _to_handle(g: Graph):
    """Host CSR handle of g (through from_edges of its u<v edges)."""
    lib = N.graph_lib()
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.offsets).astype(np.int64))
    keep = src < g.adjacency
    pairs = np.ascontiguousarray(np.stack([src[keep], g.adjacency[keep]], axis=1))
    h = ctypes.c_void_p()
    ptr = pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if pairs.size else None
    N.check_graph(lib.smg_csr_from_edges(g.n, ptr, pairs.shape[0], ctypes.byref(h), None, None))
    return h
