"""symmine on B200: a drop-in GPU engine for the reference's matching step.

The reference (arxiv 1911.12877, GraphZero; /root/reference/proj) compiles a
pattern into a nested-loop plan of ID-bounded sorted-set intersections and
differences and runs it on CPU threads (``count_instances``,
proj/src/engine.cpp:145-179).  This package keeps that plan format and the
reference's Python surface (python/symmine/__init__.py) for the matching path
and executes it with hand-written CUDA for sm_100a:

    from paper_1911_12877_b200 import Graph, named_plan, count
    g = Graph.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)])
    count(g, named_plan("triangle"))        # -> 4
"""
from ._native import CountOverflowError, InputError, IoError
from .engine import (CountResult, count, count_many, count_pattern, count_range, count_result, count_shard,
                     device_count, enumerate, motif_counts)
from .graph import Graph
from .plan import Plan, PlanLevel, compile_plan, motif_plans, named_plan

__all__ = [
    "CountOverflowError", "CountResult", "Graph", "InputError", "IoError", "Plan", "PlanLevel",
    "compile_plan", "count", "count_many", "count_pattern", "count_range", "count_result", "count_shard",
    "device_count", "enumerate", "motif_counts", "motif_plans", "named_plan",
]

__version__ = "0.1.0"
