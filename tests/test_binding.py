"""The reference-side Python binding of the drop-in (tests/cpp/pybind_count_gpu.cpp,
INTEGRATION.md): the reference's own pybind module (_core, proj/python/module.cpp
built from /root/reference by `make -C oracle pybind`) plus `symmine_gpu.count`,
which takes the reference's Graph / Plan objects and calls
symmine::gpu::count_instances.  Skipped where oracle/_ref was not built."""
from __future__ import annotations

import glob
import os
import sys

import pytest

from common import er_graph

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


@pytest.fixture(scope="module")
def mods():
    if not (glob.glob(os.path.join(REF, "_core*.so")) and glob.glob(os.path.join(REF, "symmine_gpu*.so"))):
        pytest.skip("oracle/_ref python modules not built (make -C oracle pybind)")
    sys.path.insert(0, REF)
    import _core
    import symmine_gpu
    return _core, symmine_gpu


def test_binding_shares_reference_types_and_errors(mods):
    """Host-only: the binding accepts the reference's Graph/Plan objects and its
    errors arrive as the reference's exception types (module.cpp:60-62)."""
    _core, symmine_gpu = mods
    from paper_1911_12877_b200 import engine
    g = _core.Graph.from_edges(4, [(0, 1), (1, 2), (0, 2), (2, 3)])
    p = _core.compile_plan(_core.named_pattern("triangle"))
    if engine.device_count() == 0:
        with pytest.raises(_core.IoError):  # no CPU path: IoError, an IOError
            symmine_gpu.count(g, p, 1)
    else:
        assert symmine_gpu.count(g, p, 1) == _core.count(g, p, 1) == 1
    with pytest.raises(TypeError):
        symmine_gpu.count("not a graph", p, 1)


@pytest.mark.gpu
def test_python_binding_drop_in(mods):
    _core, symmine_gpu = mods
    n, edges = er_graph(60, 0.3, 17)
    g = _core.Graph.from_edges(n, edges)
    for name in ("triangle", "rectangle", "house", "pentagon", "tailed_triangle"):
        pat = _core.named_pattern(name)
        for r, b in ((True, True), (False, True), (True, False)):
            plan = _core.compile_plan(pat, -1, r, b)
            assert symmine_gpu.count(g, plan, 1) == _core.count(g, plan, 4), (name, r, b)
    bad = _core.Plan.from_json(_core.compile_plan(_core.named_pattern("triangle")).to_json()
                               .replace('"parent":1', '"parent":2'))
    with pytest.raises(ValueError):
        symmine_gpu.count(g, bad, 1)
    symmine_gpu.release(g)
