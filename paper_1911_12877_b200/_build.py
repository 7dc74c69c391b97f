"""In-tree build of the native libraries (no JIT cache: the built .so files
travel with the repo snapshot to the GPU box).

* engine  : nvcc -gencode arch=compute_100a,code=sm_100a -> libsymmine_gpu.so
* graph   : g++ -fopenmp                                  -> libsymmine_graph.so
* oracle  : make -C oracle (test infrastructure: the C restatement always,
            the reference library only when /root/reference is present)
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
ENGINE_SO = os.path.join(PKG, "libsymmine_gpu.so")
GRAPH_SO = os.path.join(PKG, "libsymmine_graph.so")
ORACLE_DIR = os.path.join(ROOT, "oracle")
REFERENCE = "/root/reference/proj"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the CUDA engine")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _engine_headers() -> list[str]:
    return (sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(CSRC, "*.hpp"))) +
            sorted(glob.glob(os.path.join(INCLUDE, "*.h"))))


def build_engine(force: bool = False, verbose: bool = False) -> str:
    """Each .cu is compiled to an object of its own (in parallel, only when it or
    a header changed), then linked into libsymmine_gpu.so."""
    from concurrent.futures import ThreadPoolExecutor
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr = _engine_headers()
    objdir = os.path.join(CSRC, "_obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    jobs = []
    for src in cu:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, [src, *hdr]):
            cmd = [_nvcc(), *flags, "-I", INCLUDE, "-c", "-o", obj, src]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
    if jobs:
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            list(ex.map(lambda c: subprocess.run(c, check=True), jobs))
    objs = [os.path.join(objdir, os.path.basename(src)[:-3] + ".o") for src in cu]
    if force or jobs or _stale(ENGINE_SO, objs):
        tmp = ENGINE_SO + ".tmp"
        subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs],
                       check=True)
        os.replace(tmp, ENGINE_SO)
    return ENGINE_SO


def build_graph_lib(force: bool = False) -> str:
    src = os.path.join(CSRC, "graphgen.cpp")
    if force or _stale(GRAPH_SO, [src, os.path.join(INCLUDE, "symmine_graph.h")]):
        tmp = GRAPH_SO + ".tmp"
        subprocess.run(["g++", "-O3", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-Wall",
                        "-o", tmp, src], check=True)
        os.replace(tmp, GRAPH_SO)
    return GRAPH_SO


def build_oracle(reference: bool | None = None) -> None:
    """Checker libraries (test infrastructure only)."""
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, "port"], check=True)
    if reference is None:
        reference = os.path.isdir(REFERENCE)
    if reference:
        subprocess.run(["make", "-s", "-j8", "-C", ORACLE_DIR, "ref"], check=True)
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "adapter"], check=True)


def ensure_engine() -> str:
    if not os.path.exists(ENGINE_SO):
        build_engine()
    return ENGINE_SO


def ensure_graph_lib() -> str:
    if not os.path.exists(GRAPH_SO):
        build_graph_lib()
    return GRAPH_SO


def build_all(force: bool = False) -> None:
    build_engine(force)
    build_graph_lib(force)
    build_oracle()
