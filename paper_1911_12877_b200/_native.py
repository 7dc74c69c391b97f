"""ctypes bindings of the two native libraries of the package.

* ``libsymmine_gpu.so``  -- the CUDA engine behind the C ABI in
  ``include/symmine_gpu.h`` (the drop-in for ``symmine::count_instances``,
  reference proj/include/symmine/engine.hpp:23).
* ``libsymmine_graph.so`` -- the host CSR toolkit in ``include/symmine_graph.h``
  (``Graph::from_edges`` layout, seeded BASELINE generators).

There is no CPU fallback: if the engine library is missing or the machine has
no CUDA device, the count calls raise.  Libraries are built in-tree by
``_build.build_all()`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import _build

HERE = os.path.dirname(os.path.abspath(__file__))
MAX_LEVELS = 8
MAX_GPUS = 8

SMG_OK, SMG_EIO, SMG_EINPUT, SMG_EOVERFLOW = 0, 1, 2, 3
SMG_GENERIC = 2  # flag: plan executor even where a folded kernel exists
SMG_FOLDED_RANGE = 4  # flag: folded passes for root ranges of the two-centre kinds
SMG_PLAN_USE_BOUNDS = 1
SMG_PLAN_USE_RESTRICTIONS = 2
SMG_METER = 1


class InputError(ValueError):
    """Bad plan/graph input (reference InputError, error.hpp:10-12; Python
    maps it to ValueError, python/module.cpp:60)."""


class IoError(IOError):
    """CUDA/device/I-O failure (reference IoError, error.hpp:15-17)."""


class CountOverflowError(OverflowError):
    """Count exceeds 64 bits (reference CountOverflowError, error.hpp:19-22)."""


class SmgPlan(ctypes.Structure):
    _fields_ = [
        ("depth", ctypes.c_int32),
        ("isect_mask", ctypes.c_uint8 * MAX_LEVELS),
        ("diff_mask", ctypes.c_uint8 * MAX_LEVELS),
        ("parent", ctypes.c_int8 * MAX_LEVELS),
        ("flags", ctypes.c_uint32),
    ]


class SmgResult(ctypes.Structure):
    _fields_ = [
        ("count", ctypes.c_uint64),
        ("per_gpu", ctypes.c_uint64 * MAX_GPUS),
        ("elements", ctypes.c_uint64),
        ("units", ctypes.c_uint64),
        ("wall_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("count_hi", ctypes.c_int64),
    ]


_lock = threading.Lock()
_gpu = None
_graph = None

_P = ctypes.c_void_p
_U64P = ctypes.POINTER(ctypes.c_uint64)
_U32P = ctypes.POINTER(ctypes.c_uint32)


def _bind(lib, name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


def gpu_lib():
    """The CUDA engine library (built if missing; raises if it cannot be)."""
    global _gpu
    with _lock:
        if _gpu is None:
            path = _build.ensure_engine()
            lib = ctypes.CDLL(path)
            _bind(lib, "smg_abi_version", ctypes.c_int, [])
            _bind(lib, "smg_last_error", ctypes.c_char_p, [])
            _bind(lib, "smg_device_count", ctypes.c_int, [])
            _bind(lib, "smg_plan_validate", ctypes.c_int, [ctypes.POINTER(SmgPlan)])
            _bind(lib, "smg_plan_describe", ctypes.c_int,
                  [ctypes.POINTER(SmgPlan), ctypes.c_char_p, ctypes.c_size_t])
            _bind(lib, "smg_graph_create", ctypes.c_int,
                  [_U64P, _U32P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                   ctypes.POINTER(_P)])
            _bind(lib, "smg_graph_destroy", None, [_P])
            _bind(lib, "smg_graph_from_edges", ctypes.c_int,
                  [_U32P, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                   ctypes.POINTER(_P), _U64P, _U64P])
            _bind(lib, "smg_graph_orient", ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_P), _U32P])
            _bind(lib, "smg_graph_download", ctypes.c_int, [_P, ctypes.c_int, _U64P, _U32P])
            _bind(lib, "smg_enumerate", ctypes.c_int,
                  [_P, ctypes.POINTER(SmgPlan), ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _U32P,
                   ctypes.c_uint64, _U64P])
            _bind(lib, "smg_graph_set_stream", ctypes.c_int, [_P, ctypes.c_int, _P])
            _bind(lib, "smg_graph_info", ctypes.c_int,
                  [_P, _U64P, _U64P, _U64P, ctypes.POINTER(ctypes.c_int)])
            _bind(lib, "smg_count", ctypes.c_int,
                  [_P, ctypes.POINTER(SmgPlan), ctypes.c_uint, ctypes.c_uint32,
                   ctypes.POINTER(SmgResult)])
            _bind(lib, "smg_count_many", ctypes.c_int,
                  [_P, ctypes.POINTER(SmgPlan), ctypes.c_uint32, ctypes.c_uint, ctypes.c_uint32,
                   ctypes.POINTER(SmgResult)])
            _bind(lib, "smg_phase_times", ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_double)])
            _bind(lib, "smg_count_many_shard", ctypes.c_int,
                  [_P, ctypes.POINTER(SmgPlan), ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                   ctypes.c_uint32, ctypes.POINTER(SmgResult)])
            _bind(lib, "smg_count_shard", ctypes.c_int,
                  [_P, ctypes.POINTER(SmgPlan), ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                   ctypes.c_uint32, ctypes.POINTER(SmgResult)])
            _bind(lib, "smg_count_range", ctypes.c_int,
                  [_P, ctypes.POINTER(SmgPlan), ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                   ctypes.c_uint32, ctypes.POINTER(SmgResult)])
            _bind(lib, "smg_shard_bounds", ctypes.c_int,
                  [_P, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, _U64P])
            if lib.smg_abi_version() != 2:
                raise IoError("libsymmine_gpu.so ABI version mismatch; rebuild")
            _gpu = lib
        return _gpu


def graph_lib():
    """The host CSR toolkit library."""
    global _graph
    with _lock:
        if _graph is None:
            path = _build.ensure_graph_lib()
            lib = ctypes.CDLL(path)
            _bind(lib, "smg_graph_last_error", ctypes.c_char_p, [])
            _bind(lib, "smg_csr_from_edges", ctypes.c_int,
                  [ctypes.c_uint64, _U32P, ctypes.c_uint64, ctypes.POINTER(_P), _U64P, _U64P])
            _bind(lib, "smg_gen_er", ctypes.c_int,
                  [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(_P)])
            _bind(lib, "smg_gen_rmat", ctypes.c_int,
                  [ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                   ctypes.c_double, ctypes.c_uint64, ctypes.POINTER(_P)])
            _bind(lib, "smg_gen_chung_lu", ctypes.c_int,
                  [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                   ctypes.c_uint64, ctypes.POINTER(_P)])
            _bind(lib, "smg_csr_orient", ctypes.c_int, [_P, ctypes.POINTER(_P), _U32P])
            _bind(lib, "smg_csr_info", ctypes.c_int, [_P, _U64P, _U64P, _U64P])
            _bind(lib, "smg_csr_offsets", _U64P, [_P])
            _bind(lib, "smg_csr_adjacency", _U32P, [_P])
            _bind(lib, "smg_csr_free", None, [_P])
            _graph = lib
        return _graph


def raise_for(code: int, message: str) -> None:
    if code == SMG_OK:
        return
    if code == SMG_EINPUT:
        raise InputError(message)
    if code == SMG_EOVERFLOW:
        raise CountOverflowError(message)
    raise IoError(message)


def check_gpu(code: int) -> None:
    if code != SMG_OK:
        raise_for(code, gpu_lib().smg_last_error().decode())


def check_graph(code: int) -> None:
    if code != SMG_OK:
        raise_for(code, graph_lib().smg_graph_last_error().decode())
