"""Python face of the C ABI: the reference's engine entry points on B200.

    count(graph, plan, gpus=1)           ~ symmine.count(graph, plan, workers)
                                           (python/module.cpp:162-167 -> count_instances,
                                            engine.cpp:145-179)
    count_pattern(graph, name, gpus=1)   ~ symmine.count_pattern (module.cpp:168-175)
    motif_counts(graph, k, gpus=1)       ~ symmine.motif_counts (module.cpp:182-196,
                                            engine.cpp:193-205)
    count_range(graph, plan, lo, hi)     ~ Executor::count_range (engine.cpp:36-43)
    count_shard(graph, plan, shard, n)   one rank's share of the level-1 units

Every call runs on the GPU through libsymmine_gpu.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _native as N
from .graph import Graph
from .plan import Plan, motif_plans, named_plan


@dataclass
class CountResult:
    """CountResult (engine.hpp:11-15) plus device counters."""

    count: int
    per_gpu: list = field(default_factory=list)
    elements: int = 0   # E, intersected elements (meter=True only)
    units: int = 0      # level-1 partial embeddings processed
    wall_ms: float = 0.0
    kernel_ms: float = 0.0


def _result(r: N.SmgResult, ngpu: int) -> CountResult:
    # count_hi: a shard's share of a folded full count may be signed (128-bit)
    count = (int(r.count_hi) << 64) + int(r.count)
    return CountResult(count, [int(r.per_gpu[i]) for i in range(ngpu)], int(r.elements),
                       int(r.units), float(r.wall_ms), float(r.kernel_ms))


def _plan(plan) -> Plan:
    if isinstance(plan, Plan):
        return plan
    if isinstance(plan, (str, dict)):
        return Plan.from_json(plan)
    raise N.InputError("plan must be a Plan or plan JSON")


def _flags(meter: bool, generic: bool, folded: bool = False) -> int:
    return (N.SMG_METER if meter else 0) | (N.SMG_GENERIC if generic else 0) | \
        (N.SMG_FOLDED_RANGE if folded else 0)


def count_result(graph: Graph, plan, gpus: int = 1, meter: bool = False, generic: bool = False) -> CountResult:
    """count_instances(g, plan, workers=gpus) on `gpus` B200s (one process).
    generic=True forces the plan executor where a folded kernel exists."""
    p = _plan(plan)
    gpus = max(1, int(gpus))  # workers == 0 -> 1 (engine.cpp:146)
    lib = N.gpu_lib()
    h = graph.device_handle(tuple(range(gpus)))
    sp = p.to_smg()
    r = N.SmgResult()
    N.check_gpu(lib.smg_count(h, ctypes.byref(sp), gpus, _flags(meter, generic), ctypes.byref(r)))
    return _result(r, gpus)


def count(graph: Graph, plan, gpus: int = 1) -> int:
    return count_result(graph, plan, gpus).count


def count_pattern(graph: Graph, name: str, k: int = 0, gpus: int = 1) -> int:
    return count(graph, named_plan(name, k), gpus)


def count_many(graph: Graph, plans, gpus: int = 1, generic: bool = False) -> list[CountResult]:
    """One count_instances per plan, as one call (smg_count_many): work the
    plans share (the 4-clique count, triangle-per-edge and 4-cycle passes of
    the 4-vertex closed forms) is done once."""
    ps = [_plan(p) for p in plans]
    gpus = max(1, int(gpus))
    lib = N.gpu_lib()
    h = graph.device_handle(tuple(range(gpus)))
    arr = (N.SmgPlan * max(1, len(ps)))(*[p.to_smg() for p in ps])
    res = (N.SmgResult * max(1, len(ps)))()
    N.check_gpu(lib.smg_count_many(h, arr, len(ps), gpus, _flags(False, generic), res))
    return [_result(res[i], gpus) for i in range(len(ps))]


def motif_counts(graph: Graph, k: int, gpus: int = 1) -> list[dict]:
    """motif_counts (engine.cpp:193-205): every connected k-vertex pattern with
    its own plan, counted in one smg_count_many call."""
    recs = motif_plans(k)
    res = count_many(graph, [rec["plan"] for rec in recs], gpus)
    return [{"bits": rec["bits"], "name": rec["name"], "key": rec["key"], "count": r.count}
            for rec, r in zip(recs, res)]


def count_range(graph: Graph, plan, lo: int, hi: int, device: int = 0, meter: bool = False,
                generic: bool = False, folded: bool = False) -> CountResult:
    """Executor::count_range(lo, hi).  folded=True: the folded per-unit passes
    even for the two-centre kinds (default: the generic executor there)."""
    p = _plan(plan)
    lib = N.gpu_lib()
    h = graph.device_handle((device,))
    sp = p.to_smg()
    r = N.SmgResult()
    N.check_gpu(lib.smg_count_range(h, ctypes.byref(sp), 0, lo, hi, _flags(meter, generic, folded),
                                    ctypes.byref(r)))
    return _result(r, 1)


def count_shard(graph: Graph, plan, shard: int, num_shards: int, device: int = 0,
                meter: bool = False, generic: bool = False) -> CountResult:
    p = _plan(plan)
    lib = N.gpu_lib()
    h = graph.device_handle((device,))
    sp = p.to_smg()
    r = N.SmgResult()
    N.check_gpu(lib.smg_count_shard(h, ctypes.byref(sp), 0, shard, num_shards,
                                    _flags(meter, generic), ctypes.byref(r)))
    return _result(r, 1)


def enumerate(graph: Graph, plan, limit: int | None = None, device: int = 0,
              max_tuples: int = 1 << 24) -> list[tuple]:
    """symmine.enumerate (python/module.cpp:176-181 -> enumerate_instances,
    engine.cpp:181-191): embeddings as vertex tuples in the reference's order
    (level-0 ascending, then lexicographic), truncated at `limit`."""
    import numpy as np
    p = _plan(plan)
    lib = N.gpu_lib()
    h = graph.device_handle((device,))
    sp = p.to_smg()
    cap = max_tuples if limit is None else min(limit, max_tuples)
    out = np.zeros(max(cap, 1) * sp.depth, dtype=np.uint32)
    n_out = ctypes.c_uint64()
    N.check_gpu(lib.smg_enumerate(h, ctypes.byref(sp), 0, limit is not None,
                                  0 if limit is None else limit,
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), cap,
                                  ctypes.byref(n_out)))
    if n_out.value > cap:
        raise N.InputError(f"{n_out.value} embeddings exceed max_tuples={max_tuples}")
    rows = out[: n_out.value * sp.depth].reshape(-1, sp.depth)
    return [tuple(int(x) for x in r) for r in rows]


def device_count() -> int:
    return int(N.gpu_lib().smg_device_count())
