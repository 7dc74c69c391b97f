"""TEST INFRASTRUCTURE ONLY: ctypes access to the checkers.

* ``Reference`` -- the reference symmine library compiled from
  /root/reference (oracle/_ref/libsymmine_ref.so, see oracle/Makefile and
  ref_shim.cpp).  Present only where it was built (this container, or a GPU
  box that received the prebuilt file).
* ``Port``      -- the plain-C restatement (oracle/_build/liboracle.so,
  symmine_oracle.c), always buildable with gcc.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsymmine_ref.so")
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")

_P = ctypes.c_void_p
_U64P = ctypes.POINTER(ctypes.c_uint64)
_U32P = ctypes.POINTER(ctypes.c_uint32)


def _u64(a):
    return a.ctypes.data_as(_U64P)


def _u32(a):
    return a.ctypes.data_as(_U32P)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _bind(lib, name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The reference engine itself (compiled from /root/reference)."""

    _lib = None

    def __init__(self):
        if Reference._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO)
            lib = ctypes.CDLL(REF_SO)
            _bind(lib, "ref_last_error", ctypes.c_char_p, [])
            _bind(lib, "ref_graph_from_edges", _P, [ctypes.c_uint64, _U32P, ctypes.c_uint64, _U64P, _U64P])
            _bind(lib, "ref_graph_free", None, [_P])
            _bind(lib, "ref_graph_shape", None, [_P, _U64P, _U64P, _U64P])
            _bind(lib, "ref_graph_csr", None, [_P, _U64P, _U32P])
            _bind(lib, "ref_graph_orient", _P, [_P, _U32P])
            _bind(lib, "ref_plan_json", ctypes.c_int,
                  [ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                   ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t])
            _bind(lib, "ref_motif_plans_json", ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t])
            _bind(lib, "ref_plan_from_json", _P, [ctypes.c_char_p])
            _bind(lib, "ref_plan_free", None, [_P])
            _bind(lib, "ref_count", ctypes.c_int, [_P, _P, ctypes.c_uint, _U64P, ctypes.POINTER(ctypes.c_double)])
            _bind(lib, "ref_count_range", ctypes.c_int, [_P, _P, ctypes.c_uint32, ctypes.c_uint32, _U64P])
            _bind(lib, "ref_enumerate", ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_uint64, _U32P, ctypes.c_uint64, _U64P])
            _bind(lib, "ref_count_chunks", ctypes.c_int,
                  [_P, _P, ctypes.c_uint, _U32P, ctypes.c_uint64, _U64P, _U64P, ctypes.POINTER(ctypes.c_uint8)])
            _bind(lib, "ref_count_roots", ctypes.c_int,
                  [_P, _P, ctypes.c_uint, _U32P, ctypes.c_uint64, _U64P, _U64P])
            _bind(lib, "ref_count_units", ctypes.c_int,
                  [_P, _P, ctypes.c_uint, _U32P, _U32P, ctypes.c_uint64, _U64P, _U64P, ctypes.c_double, _U64P])
            _bind(lib, "ref_oracle_induced", ctypes.c_int,
                  [_P, ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, _U64P])
            Reference._lib = lib
        self.lib = Reference._lib

    def _err(self, code):
        raise OracleError(code, self.lib.ref_last_error().decode())

    # --- plans -----------------------------------------------------------
    def plan_json(self, name="", k=0, pattern_text=None, schedule_index=-1,
                  use_restrictions=True, use_bounds=True) -> dict:
        cap = 1 << 16
        buf = ctypes.create_string_buffer(cap)
        rc = self.lib.ref_plan_json(name.encode(), k, (pattern_text or "").encode(), schedule_index,
                                    int(use_restrictions), int(use_bounds), buf, cap)
        if rc:
            self._err(rc)
        return json.loads(buf.value.decode())

    def motif_plans(self, k) -> list:
        cap = 1 << 22
        buf = ctypes.create_string_buffer(cap)
        rc = self.lib.ref_motif_plans_json(k, buf, cap)
        if rc:
            self._err(rc)
        return json.loads(buf.value.decode())

    # --- graphs ----------------------------------------------------------
    def graph_from_edges(self, n, pairs):
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
        d = ctypes.c_uint64()
        s = ctypes.c_uint64()
        h = self.lib.ref_graph_from_edges(n, _u32(pairs), pairs.shape[0], ctypes.byref(d), ctypes.byref(s))
        if not h:
            self._err(2)
        return RefGraph(self, h), d.value, s.value

    def graph_from_csr(self, off, adj):
        off = np.asarray(off, dtype=np.uint64)
        adj = np.asarray(adj, dtype=np.uint32)
        n = len(off) - 1
        src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(off).astype(np.int64))
        keep = src < adj
        pairs = np.stack([src[keep], adj[keep]], axis=1)
        g, _, _ = self.graph_from_edges(n, pairs)
        return g


class RefGraph:
    def __init__(self, ref, handle):
        self.ref = ref
        self.h = handle

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    def csr(self):
        n, s, m = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self.ref.lib.ref_graph_shape(self.h, ctypes.byref(n), ctypes.byref(s), ctypes.byref(m))
        off = np.zeros(n.value + 1, dtype=np.uint64)
        adj = np.zeros(max(s.value, 1), dtype=np.uint32)
        self.ref.lib.ref_graph_csr(self.h, _u64(off), _u32(adj))
        return off, adj[: s.value]

    def orient(self):
        n = len(self.csr()[0]) - 1
        new_to_old = np.zeros(max(n, 1), dtype=np.uint32)
        h = self.ref.lib.ref_graph_orient(self.h, _u32(new_to_old))
        return RefGraph(self.ref, h), new_to_old[:n]

    def _plan(self, plan_json):
        text = plan_json if isinstance(plan_json, str) else json.dumps(plan_json)
        p = self.ref.lib.ref_plan_from_json(text.encode())
        if not p:
            self.ref._err(2)
        return p

    def count(self, plan_json, workers=1):
        p = self._plan(plan_json)
        try:
            c = ctypes.c_uint64()
            ms = ctypes.c_double()
            rc = self.ref.lib.ref_count(self.h, p, workers, ctypes.byref(c), ctypes.byref(ms))
            if rc:
                self.ref._err(rc)
            return c.value, ms.value
        finally:
            self.ref.lib.ref_plan_free(p)

    def count_range(self, plan_json, lo, hi):
        p = self._plan(plan_json)
        try:
            c = ctypes.c_uint64()
            rc = self.ref.lib.ref_count_range(self.h, p, lo, hi, ctypes.byref(c))
            if rc:
                self.ref._err(rc)
            return c.value
        finally:
            self.ref.lib.ref_plan_free(p)

    def count_chunks(self, plan_json, starts, order, counts, done, workers):
        """Dynamic root-chunk queue (one Executor per thread); fills counts/done
        in place so a caller thread can checkpoint while it runs."""
        p = self._plan(plan_json)
        try:
            starts = np.ascontiguousarray(starts, dtype=np.uint32)
            order = np.ascontiguousarray(order, dtype=np.uint64)
            rc = self.ref.lib.ref_count_chunks(self.h, p, workers, _u32(starts), len(starts) - 1, _u64(order),
                                               _u64(counts), done.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
            if rc:
                self.ref._err(rc)
        finally:
            self.ref.lib.ref_plan_free(p)

    def count_roots(self, plan_json, roots, workers):
        """Per-root counts and per-root CPU ns (dynamic queue, one Executor per thread)."""
        p = self._plan(plan_json)
        try:
            roots = np.ascontiguousarray(roots, dtype=np.uint32)
            counts = np.zeros(max(len(roots), 1), dtype=np.uint64)
            ns = np.zeros(max(len(roots), 1), dtype=np.uint64)
            rc = self.ref.lib.ref_count_roots(self.h, p, workers, _u32(roots), len(roots), _u64(counts), _u64(ns))
            if rc:
                self.ref._err(rc)
            return counts[: len(roots)], ns[: len(roots)]
        finally:
            self.ref.lib.ref_plan_free(p)

    def count_units(self, plan_json, v0, v1, workers, budget_s=0.0):
        """Per-unit counts of level-1 units (v0, v1) (the reference's count_from(2))
        and per-unit CPU ns; dynamic queue, one Executor per thread.  With a
        budget, only a prefix of the units is counted: the returned arrays are
        cut to it."""
        p = self._plan(plan_json)
        try:
            v0 = np.ascontiguousarray(v0, dtype=np.uint32)
            v1 = np.ascontiguousarray(v1, dtype=np.uint32)
            counts = np.zeros(max(len(v0), 1), dtype=np.uint64)
            ns = np.zeros(max(len(v0), 1), dtype=np.uint64)
            done = ctypes.c_uint64()
            rc = self.ref.lib.ref_count_units(self.h, p, workers, _u32(v0), _u32(v1), len(v0), _u64(counts),
                                              _u64(ns), float(budget_s), ctypes.byref(done))
            if rc:
                self.ref._err(rc)
            return counts[: done.value], ns[: done.value]
        finally:
            self.ref.lib.ref_plan_free(p)

    def enumerate(self, plan_json, limit=None):
        p = self._plan(plan_json)
        try:
            depth = len(json.loads(plan_json)["levels"]) if isinstance(plan_json, str) else len(plan_json["levels"])
            cap = 1 << 20
            out = np.zeros(cap * depth, dtype=np.uint32)
            n = ctypes.c_uint64()
            rc = self.ref.lib.ref_enumerate(self.h, p, limit is not None, 0 if limit is None else limit, _u32(out), cap,
                                            ctypes.byref(n))
            if rc:
                self.ref._err(rc)
            if limit == 0:
                return []
            k = min(n.value, cap)
            return [tuple(int(x) for x in out[i * depth:(i + 1) * depth]) for i in range(k)]
        finally:
            self.ref.lib.ref_plan_free(p)

    def oracle_induced(self, name="", k=0, pattern_text=None):
        c = ctypes.c_uint64()
        rc = self.ref.lib.ref_oracle_induced(self.h, name.encode(), k, (pattern_text or "").encode(),
                                             ctypes.byref(c))
        if rc:
            self.ref._err(rc)
        return c.value


class Port:
    """The plain-C restatement (symmine_oracle.c)."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            if not os.path.exists(PORT_SO):
                subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
            lib = ctypes.CDLL(PORT_SO)
            from paper_1911_12877_b200._native import SmgPlan  # POD struct only
            self.SmgPlan = SmgPlan
            pp = ctypes.POINTER(SmgPlan)
            _bind(lib, "oracle_intersect", ctypes.c_size_t,
                  [_U32P, ctypes.c_size_t, _U32P, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32, _U32P])
            _bind(lib, "oracle_difference", ctypes.c_size_t,
                  [_U32P, ctypes.c_size_t, _U32P, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32, _U32P])
            _bind(lib, "oracle_count_range", ctypes.c_int,
                  [_U64P, _U32P, ctypes.c_uint64, pp, ctypes.c_uint32, ctypes.c_uint32, _U64P, _U64P])
            _bind(lib, "oracle_count", ctypes.c_int,
                  [_U64P, _U32P, ctypes.c_uint64, pp, ctypes.c_int, _U64P, _U64P])
            _bind(lib, "oracle_count_edges", ctypes.c_int,
                  [_U64P, _U32P, ctypes.c_uint64, pp, _U64P, ctypes.c_uint64, _U64P, _U64P])
            _bind(lib, "oracle_enumerate", ctypes.c_int,
                  [_U64P, _U32P, ctypes.c_uint64, pp, ctypes.c_uint64, _U32P, _U64P])
            _bind(lib, "oracle_from_edges", ctypes.c_int,
                  [ctypes.c_uint64, _U32P, ctypes.c_uint64, _U64P, _U32P, _U64P, _U64P, _U64P])
            _bind(lib, "oracle_orient", ctypes.c_int, [_U64P, _U32P, ctypes.c_uint64, _U64P, _U32P, _U32P])
            Port._lib = lib
        self.lib = Port._lib

    @staticmethod
    def _csr(off, adj):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        if adj.size == 0:
            adj = np.zeros(1, dtype=np.uint32)
        return off, adj

    def intersect(self, a, b, bound=None):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros(max(len(a), 1), dtype=np.uint32)
        k = self.lib.oracle_intersect(_u32(a), len(a), _u32(b), len(b), bound is not None,
                                      0 if bound is None else bound, _u32(out))
        return out[:k].tolist()

    def difference(self, a, b, bound=None):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros(max(len(a), 1), dtype=np.uint32)
        k = self.lib.oracle_difference(_u32(a), len(a), _u32(b), len(b), bound is not None,
                                       0 if bound is None else bound, _u32(out))
        return out[:k].tolist()

    def count_range(self, off, adj, smg_plan, lo, hi):
        off, adj = self._csr(off, adj)
        c, e = ctypes.c_uint64(), ctypes.c_uint64()
        rc = self.lib.oracle_count_range(_u64(off), _u32(adj), len(off) - 1, ctypes.byref(smg_plan),
                                         lo, hi, ctypes.byref(c), ctypes.byref(e))
        if rc:
            raise OracleError(rc, "oracle_count_range failed")
        return c.value, e.value

    def count(self, off, adj, smg_plan, threads=1):
        off, adj = self._csr(off, adj)
        c, e = ctypes.c_uint64(), ctypes.c_uint64()
        rc = self.lib.oracle_count(_u64(off), _u32(adj), len(off) - 1, ctypes.byref(smg_plan), threads,
                                   ctypes.byref(c), ctypes.byref(e))
        if rc:
            raise OracleError(rc, "oracle_count failed")
        return c.value, e.value

    def count_edges(self, off, adj, smg_plan, slots):
        off, adj = self._csr(off, adj)
        slots = np.ascontiguousarray(slots, dtype=np.uint64)
        c, e = ctypes.c_uint64(), ctypes.c_uint64()
        rc = self.lib.oracle_count_edges(_u64(off), _u32(adj), len(off) - 1, ctypes.byref(smg_plan),
                                         _u64(slots), len(slots), ctypes.byref(c), ctypes.byref(e))
        if rc:
            raise OracleError(rc, "oracle_count_edges failed")
        return c.value, e.value

    def enumerate(self, off, adj, smg_plan, limit=None, cap=1 << 20):
        off, adj = self._csr(off, adj)
        depth = smg_plan.depth
        lim = 0 if limit is None else limit
        if limit == 0:
            return []
        out = np.zeros(cap * depth, dtype=np.uint32)
        n = ctypes.c_uint64()
        rc = self.lib.oracle_enumerate(_u64(off), _u32(adj), len(off) - 1, ctypes.byref(smg_plan),
                                       lim if lim else cap, _u32(out), ctypes.byref(n))
        if rc:
            raise OracleError(rc, "oracle_enumerate failed")
        return [tuple(int(x) for x in out[i * depth:(i + 1) * depth]) for i in range(n.value)]

    def from_edges(self, n, pairs):
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
        m = pairs.shape[0]
        off = np.zeros(n + 1, dtype=np.uint64)
        adj = np.zeros(max(2 * m, 1), dtype=np.uint32)
        s, d, l = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        p = pairs if m else np.zeros((1, 2), dtype=np.uint32)
        rc = self.lib.oracle_from_edges(n, _u32(p), m, _u64(off), _u32(adj), ctypes.byref(s),
                                        ctypes.byref(d), ctypes.byref(l))
        if rc:
            raise OracleError(rc, "edge endpoint out of range")
        return off, adj[: s.value], d.value, l.value

    def orient(self, off, adj):
        off, adj = self._csr(off, adj)
        n = len(off) - 1
        off2 = np.zeros(n + 1, dtype=np.uint64)
        adj2 = np.zeros(len(adj), dtype=np.uint32)
        n2o = np.zeros(max(n, 1), dtype=np.uint32)
        self.lib.oracle_orient(_u64(off), _u32(adj), n, _u64(off2), _u32(adj2), _u32(n2o))
        return off2, adj2[: int(off[-1])], n2o[:n]
