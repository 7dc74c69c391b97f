#!/usr/bin/env python
"""Benchmark: BASELINE config 2 (RMAT scale 20, edge factor 16) -- 4-clique and
induced 4-cycle counts -- on N B200s, one process per GPU.

Metric (BASELINE.json): pattern count time and intersected elements/s, exact
counts.  One step = counting both patterns over the resident graph (each rank
its shard of the level-1 edge units, then one NCCL allreduce of the uint64
counters).  `value` = E_total / step time (E = intersected elements, SURVEY
8(d), measured once by the engine's metering pass; it is a property of graph +
plan).  `e2e` = the same through the public API from pinned host buffers
(graph upload + count + result read-back every step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "cfg2"
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2
CPU_SAMPLE_SECONDS = float(os.environ.get("SMG_CPU_SAMPLE_S", "15"))


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxs.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxs),
                "reasons": sorted(reasons), "samples": len(sms)}


# -------------------------------------------------------------- CPU legs ---
def unit_sample(offsets, adjacency, plan, size, seed):
    """Uniform edge-slot sample of the plan's level-1 units (v0, v1): slots drawn
    without replacement from those passing level 1's bound (the
    better estimator; hubs included at their edge share)."""
    import numpy as np
    deg = np.diff(offsets.astype(np.int64))
    src = np.repeat(np.arange(deg.size, dtype=np.uint32), deg)
    ok = np.ones(adjacency.size, dtype=bool)
    if plan.to_smg().parent[1] == 0:
        ok = adjacency < src
    pool = np.flatnonzero(ok)
    rng = np.random.default_rng(seed)
    pick = rng.choice(pool, size=min(size, pool.size), replace=False)
    return pick.astype(np.uint64), src[pick], adjacency[pick]


def sample_elements(offsets, adjacency, plan, slots, threads):
    """E of the sampled units from the C restatement's meter (untimed)."""
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    from oracle.ref import Port
    port = Port()
    sp = plan.to_smg()
    parts = np.array_split(np.asarray(slots, dtype=np.uint64), max(1, threads * 4))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return sum(ex.map(lambda s: port.count_edges(offsets, adjacency, sp, s)[1] if s.size else 0, parts))


class CpuReference:
    """The reference's own CPU engine (oracle/_ref, compiled from
    /root/reference): Executor::count_from(2) per level-1 unit (the exact path
    count_range runs for it, engine.cpp:36-43, 89-115), one Executor per host
    thread, one continuous dynamic queue over the sample.  Falls back to the C
    restatement's threaded per-unit counts when the reference library is
    absent (kind "port")."""

    def __init__(self, offsets, adjacency, plans, threads):
        from oracle.ref import Port, Reference, reference_available
        self.off, self.adj, self.plans, self.threads = offsets, adjacency, plans, threads
        self.kind = "reference" if reference_available() else "port"
        if self.kind == "reference":
            self.rg = Reference().graph_from_csr(offsets, adjacency)
        else:
            self.port = Port()

    def run(self, plan, slots, v0, v1, budget_s=0.0):
        """Count the units (a prefix of them when budget_s > 0); returns
        (number counted, their total count, wall seconds)."""
        import numpy as np
        t0 = time.perf_counter()
        if self.kind == "reference":
            c, _ = self.rg.count_units(plan.to_json(), v0, v1, self.threads, budget_s)
            k, total = len(c), int(c.sum(dtype=np.uint64))
        else:
            from concurrent.futures import ThreadPoolExecutor
            sp = plan.to_smg()
            parts = np.array_split(slots, max(1, self.threads * 8))
            with ThreadPoolExecutor(max_workers=self.threads) as ex:
                res = list(ex.map(lambda s: self.port.count_edges(self.off, self.adj, sp, s)[0] if s.size else 0,
                                  parts))
            k, total = len(slots), sum(res)
        return k, total, time.perf_counter() - t0


def cpu_sample(graph, plans, seconds, threads, seed=2024):
    """Calibrate a bounded CPU sample of the workload: per plan, uniformly drawn
    level-1 units counted by the reference engine on all host threads until
    seconds/len(plans) elapse.  Returns (E/s, info) with the fixed sample."""
    cpu = CpuReference(graph.offsets, graph.adjacency, plans, threads)
    per = seconds / max(1, len(plans))
    sample, E, elapsed = [], 0, 0.0
    for i, (label, plan) in enumerate(plans):
        slots, v0, v1 = unit_sample(graph.offsets, graph.adjacency, plan, 1 << 21, seed + i)
        k, _, dt = cpu.run(plan, slots, v0, v1, budget_s=per)
        e = sample_elements(graph.offsets, graph.adjacency, plan, slots[:k], threads)
        sample.append((label, plan, slots[:k], v0[:k], v1[:k], e))
        E += e
        elapsed += dt
    return E / elapsed, {"kind": cpu.kind, "cores": threads, "elapsed_s": elapsed, "E": E, "cpu": cpu,
                         "sample": sample, "units": sum(len(x[2]) for x in sample)}


def estimate_full_seconds(graph, info):
    """Reference count time of the whole config, estimated from the uniform
    unit sample: per plan, sample seconds x (level-1 units of the plan / units
    sampled)."""
    import numpy as np
    deg = np.diff(graph.offsets.astype(np.int64))
    src = np.repeat(np.arange(deg.size, dtype=np.uint32), deg)
    bounded = int((graph.adjacency < src).sum())
    est = 0.0
    for label, plan, slots, v0, v1, _ in info["sample"]:
        total_units = bounded if plan.to_smg().parent[1] == 0 else graph.adjacency.size
        est += info["cpu"].run(plan, slots, v0, v1)[2] * total_units / max(1, len(slots))
    return est


def load_graph_file(cfg):
    """The config's CSR for the reference arm, read from the .npz cache with
    numpy only.  A cache miss is filled by a separate process (the seeded
    generator of paper_1911_12877_b200.configs), so no library of this repo is
    mapped into the reference arm's process."""
    import numpy as np
    from types import SimpleNamespace
    code = ("import sys; sys.path.insert(0, %r); from paper_1911_12877_b200 import configs; "
            "print(configs.cache_path(%r, fill=True))" % (ROOT, cfg))
    path = subprocess.run([sys.executable, "-c", code], check=True, capture_output=True,
                          text=True).stdout.strip().splitlines()[-1]
    z = np.load(path)
    off, adj = z["offsets"], z["adjacency"]
    return SimpleNamespace(offsets=off, adjacency=adj, n=off.size - 1, m=adj.size // 2)


def plan_list(cfg):
    """(label, plan) of the config's patterns that finish (configs.NOT_FINISHED
    names the rest; the line reports them)."""
    from paper_1911_12877_b200 import configs  # plans + descriptions only: maps no native library
    skip = configs.NOT_FINISHED.get(cfg, ())
    return [(lbl, p) for lbl, p in configs.config_patterns(cfg) if lbl not in skip]


def describe(cfg):
    from paper_1911_12877_b200 import configs
    return configs.describe(cfg)


def reference_arm(args):
    """--impl reference: the reference's own CPU engine on this box's host cores."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    graph = load_graph_file(CONFIG)
    plans = plan_list(CONFIG)
    threads = os.cpu_count() or 1
    # fix the sample once (calibration ~ one step's budget), then time K steps on it
    step_budget = float(os.environ.get("SMG_REF_STEP_S", "10"))
    _, info = cpu_sample(graph, plans, step_budget, threads)
    cpu = info["cpu"]
    times = []
    for s in range(args.warmup + args.steps):
        dt = 0.0
        for label, plan, slots, v0, v1, _ in info["sample"]:
            dt += cpu.run(plan, slots, v0, v1)[2]
        if s >= args.warmup:
            times.append(dt)
    t = sum(times)
    metered = CONFIG in METERED_CONFIGS
    if metered:
        value, metric, unit = info["E"] * len(times) / t, "intersected_elements_per_s", "elements/s"
    else:
        est = estimate_full_seconds(graph, info)
        value, metric, unit = est, "pattern_count_time_s", "s"
    sample = (f"{info['units']} level-1 units drawn uniformly over the edge slots of {CONFIG} "
              f"({', '.join(f'{lbl}: {len(sl)}' for lbl, _, sl, _, _, _ in info['sample'])}), each counted "
              f"by the reference's Executor::count_from(2) on a dynamic queue over {threads} threads")
    line = {
        "impl": "reference", "metric": metric, "value": value,
        "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / len(times), "higher_is_better": metered, "scaling": "strong",
        "estimated_from_sample": not metered,
        "vs_baseline": None, "dtype": "u32", "data": f"synthetic ({CONFIG}, seeded)",
        "config": {"workload": f"{CONFIG}: {describe(CONFIG)} (unit sample)",
                   "patterns": [lbl for lbl, _ in plans], "sample_units": info["units"]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": info["kind"],
                         "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm ---
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_profile(cfg, kernel):
    """ncu figures (DRAM bytes per step, L2 hit rate) of one kernel of this
    config's step, from the committed summary (profiles/ncu_summary.json,
    written by tools/traffic_summary.py).  The c4 phase sums c4_kernel and the
    c4_hub_kernel / c4_group_kernel launches."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    ent = d.get("workloads", {}).get(f"{cfg}:step")
    if not ent:
        return None
    per = ent.get("per_kernel", {})
    names = {"c4_kernel": ["c4_kernel", "c4_hub_kernel", "c4_group_kernel"],
             "k4_cta_kernel": ["k4_cta_kernel", "k4_warp_kernel", "count_kernel", "heavy_kernel"]}.get(kernel, [kernel])
    hit = [per[n] for n in names if n in per]
    if not hit:
        return None
    l2b = sum(p["l2_bytes"] for p in hit)
    out = {"dram_bytes": sum(p["dram_bytes"] for p in hit),
           "l2_hit_pct": (sum((p["l2_hit_pct"] or 0) * p["l2_bytes"] for p in hit) / l2b) if l2b else None,
           "launches": sum(p["launches"] for p in hit), "source": ent.get("source")}
    for k in ("sm_throughput_pct", "l2_throughput_pct", "warps_active_pct", "full_capture"):
        for p in hit:
            if k in p:
                out[k] = p[k]  # from the ncu --set full capture of the phase's main kernel
                break
    return out


# kernels one full count launches: the generic executor runs count_kernel (+
# heavy_kernel for batched leaves); tailed diamond a runs one folded kernel
# (tindex.cu); house and tailed diamond b a centre-table pass and an
# ego-network pass; the 4-vertex kinds (star4 1, tailed triangle 5, diamond 6,
# path4 7, rectangle 8/9) the 4-clique count_kernel + m4_edge_kernel
# (+ m4_vertex_kernel for 1, 5, 7; + c4_kernel for 7, 8, 9).  The triangle
# index, K5 and the k4 pair sum are built once per graph (cached).
FOLDED_LAUNCHES = {1: 3, 2: 1, 3: 2, 4: 2, 5: 3, 6: 2, 7: 4, 8: 3, 9: 3}
# configs whose E (intersected elements) the generic executor's
# metering pass measures in seconds; the others report count time only
METERED_CONFIGS = ("cfg1", "cfg2")


def launches_per_step(cfg, plans):
    """Kernel launches of one step: counted by ncu for this config's step when
    the committed summary has it (profiles/ncu_summary.json), else the sum of
    the per-count figures above."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            per = json.load(f)["workloads"][f"{cfg}:step"]["per_kernel"]
        return sum(int(p["launches"]) for p in per.values())
    except Exception:
        return sum(kernels_per_count(p)[0] for _, p in plans)


def kernels_per_count(plan):
    """(kernel launches per count, folded kind or 0)."""
    import ctypes
    from paper_1911_12877_b200 import _native as N
    sp = plan.to_smg()
    buf = ctypes.create_string_buffer(1 << 16)
    N.check_gpu(N.gpu_lib().smg_plan_describe(ctypes.byref(sp), buf, 1 << 16))
    d = json.loads(buf.value.decode())
    if d.get("fast"):
        return FOLDED_LAUNCHES[d["fast"]], d["fast"]
    return (2 if d["batch"] else 1), 0


def our_arm(args):
    import ctypes
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_12877_b200 as smg
    from paper_1911_12877_b200 import _native as N
    from paper_1911_12877_b200 import configs
    from paper_1911_12877_b200.distributed import allreduce_u64

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", rank)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator / transport lines on stderr
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum_u64(vals):
        return vals if world == 1 else allreduce_u64(vals, device=dev)

    if rank == 0:
        graph = configs.load(CONFIG, verbose=True)
    barrier()
    if rank != 0:
        graph = configs.load(CONFIG)
    plans = plan_list(CONFIG)
    lib = N.gpu_lib()
    stream = torch.cuda.current_stream(dev)
    h = graph.device_handle((local,))
    N.check_gpu(lib.smg_graph_set_stream(h, 0, ctypes.c_void_p(stream.cuda_stream)))

    def shard(plan, meter=False):
        sp = plan.to_smg()
        r = N.SmgResult()
        N.check_gpu(lib.smg_count_shard(h, ctypes.byref(sp), 0, rank, world,
                                        N.SMG_METER if meter else 0, ctypes.byref(r)))
        return r

    plan_arr = (N.SmgPlan * len(plans))(*[p.to_smg() for _, p in plans])

    def step(handle):
        """One step: this rank's shard of every pattern of the config, one
        smg_count_many_shard call (work the plans share is done once per call)."""
        res = (N.SmgResult * len(plans))()
        N.check_gpu(lib.smg_count_many_shard(handle, plan_arr, len(plans), 0, rank, world, 0, res))
        return res

    # metering pass: E per pattern (deterministic property of graph + plan).
    # Plans that lower to a folded closed-form kernel (csrc/tindex.cu) never
    # enumerate the merges E counts; a config with one reports count time.
    folded = {label: kernels_per_count(plan)[1] for label, plan in plans}
    metered = CONFIG in METERED_CONFIGS  # SMG_METER runs the generic executor
    E, counts = {}, {}
    if metered:
        for label, plan in plans:
            r = shard(plan, meter=True)
            c, e = allsum_u64([(int(r.count_hi) << 64) + int(r.count), r.elements])
            E[label], counts[label] = e, c
    else:  # count-time configs: the reference counts are the first step's (untimed)
        res0 = step(h)
        tot = allsum_u64([(int(res0[i].count_hi) << 64) + int(res0[i].count) for i in range(len(plans))])
        for (label, _), c in zip(plans, tot):
            E[label], counts[label] = None, c
    E_total = sum(E.values()) if metered else None

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ms = {label: [] for label, _ in plans}
    phase_ms = [[], [], [], []]  # per timed step: 4-clique count (k4.cu), c4 pass, edge pass, vertex pass
    for _ in range(args.warmup if metered else max(0, args.warmup - 1)):  # the count pass above warmed one
        step(h)
        flush.add_(1)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    step_counts = []
    with ClockSampler(local) as clocks:
        for s in range(args.steps):
            flush.add_(1)  # L2 flush between timed steps (outside the events)
            ev[s][0].record(stream)
            res = step(h)
            cs = [(int(res[i].count_hi) << 64) + int(res[i].count) for i in range(len(plans))]
            for i, (label, _) in enumerate(plans):
                kern_ms[label].append(res[i].kernel_ms)
            ev[s][1].record(stream)
            ph = (ctypes.c_double * 4)()
            N.check_gpu(lib.smg_phase_times(h, 0, ph))
            for q in range(4):
                phase_ms[q].append(ph[q])
            step_counts.append(cs)
        torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    t_local = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    t_step = allmax(t_local) / args.steps
    # every timed step must reproduce the metered counts
    for cs in step_counts:
        tot = allsum_u64(cs)
        assert tot == [counts[lbl] for lbl, _ in plans], (tot, counts)
    value = E_total / t_step if metered else t_step

    # ---- e2e: public C-ABI path from pinned host buffers, every step ------
    off_pin = torch.from_numpy(graph.offsets.view(np.int64)).pin_memory()
    adj_pin = torch.from_numpy(graph.adjacency.view(np.int32)).pin_memory()
    h2d = off_pin.numel() * 8 + adj_pin.numel() * 4
    d2h = 48 * len(plans)
    e2e_steps = max(1, min(args.steps, 8))
    t_e2e = 0.0
    e2e_parts = {"graph_create_ms": 0.0, "count_ms": 0.0, "graph_destroy_ms": 0.0}
    # the first iteration warms the allocator / context and is not timed, unless a
    # step takes minutes (then one iteration, timed, is all the budget allows)
    e2e_warm = 0 if t_step > 30.0 else 1
    if not e2e_warm:
        e2e_steps = 1
    for s in range(e2e_steps + e2e_warm):
        barrier()
        t0 = time.perf_counter()
        gh = ctypes.c_void_p()
        dev_arr = (ctypes.c_int * 1)(local)
        N.check_gpu(lib.smg_graph_create(ctypes.cast(off_pin.data_ptr(), ctypes.POINTER(ctypes.c_uint64)),
                                         ctypes.cast(adj_pin.data_ptr(), ctypes.POINTER(ctypes.c_uint32)),
                                         graph.n, dev_arr, 1, ctypes.byref(gh)))
        t1 = time.perf_counter()
        res = step(gh)
        cs = [int(res[i].count) for i in range(len(plans))]
        t2 = time.perf_counter()
        lib.smg_graph_destroy(gh)
        t3 = time.perf_counter()
        if s >= e2e_warm:
            t_e2e += t3 - t0
            for k, v in zip(e2e_parts, (t1 - t0, t2 - t1, t3 - t2)):
                e2e_parts[k] += 1e3 * v / e2e_steps
    t_e2e = allmax(t_e2e) / e2e_steps
    e2e_value = E_total / t_e2e if metered else t_e2e

    # ---- roofline of the dominant kernel (rank 0's shard) --------------------
    # Physical: the kernel's DRAM bytes per step (dram__bytes_read + write of one
    # ncu capture of this step, committed under profiles/) / its live device
    # time per step (CUDA events on the launching stream, smg_phase_times or
    # the count's kernel_ms) / the measured HBM peak.  Algorithmic: 4 B x E
    # (the bytes a merge engine would stream) / the step's kernel
    # time -- reported separately, it is not a roofline of this engine.
    step_kernel_ms = sum(statistics.mean(v) for v in kern_ms.values())
    alg_gbs = 4.0 * E_total / (step_kernel_ms / 1e3) / 1e9 if metered and world == 1 else None
    peak, peak_kind = load_peaks()
    phase_names = ["k4_cta_kernel", "c4_kernel", "m4_edge_kernel", "m4_vertex_kernel"]
    if any(statistics.mean(v) > 0 for v in phase_ms):
        kernel_ms = {nm: statistics.mean(v) for nm, v in zip(phase_names, phase_ms)}
    else:  # no closed-form batch in this config: one kernel_ms per count
        kernel_ms = {f"{lbl} (all kernels of the count)": statistics.mean(v) for lbl, v in kern_ms.items()}
    dom = max(kernel_ms, key=kernel_ms.get)
    dom_ms = kernel_ms[dom]
    prof = load_profile(CONFIG, dom)
    traffic = prof.get("dram_bytes") if prof else None
    achieved = traffic / (dom_ms / 1e3) / 1e9 if traffic else None
    frac = (achieved / peak) if achieved else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_v, info = cpu_sample(graph, plans, CPU_SAMPLE_SECONDS, os.cpu_count() or 1)
        cpu = {"value": cpu_v, "unit": "elements/s", "cores": info["cores"], "kind": info["kind"],
               "sample": (f"{info['units']} level-1 units drawn uniformly over the edge slots of {CONFIG} "
                          f"({', '.join(f'{lbl}: {len(sl)}' for lbl, _, sl, _, _, _ in info['sample'])}), "
                          f"counted by the reference's Executor::count_from(2) on one dynamic queue over "
                          f"{info['cores']} threads in {info['elapsed_s']:.1f} s; E of the sample from the "
                          f"oracle meter (untimed)")}
    if rank == 0:
        metric, unit = (("intersected_elements_per_s", "elements/s") if metered else
                        ("pattern_count_time_s", "s"))
        if cpu and not metered:
            cpu["value"], cpu["unit"] = estimate_full_seconds(graph, info), "s"
            cpu["note"] = ("reference count time of the whole config estimated from the unit sample "
                           "(sample seconds x units / units sampled)")
        line = {
            "metric": metric, "value": value, "unit": unit,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": metered, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32",
            "data": f"synthetic ({configs.describe(CONFIG)}; seeded, no public dataset named)",
            "config": {"workload": f"{CONFIG}: {configs.describe(CONFIG)} (n={graph.n}, m={graph.m})",
                       "patterns": [lbl for lbl, _ in plans], "counts": counts,
                       "patterns_not_finished": list(configs.NOT_FINISHED.get(CONFIG, ())),
                       "elements": E, "pattern_ms": {k: statistics.mean(v) for k, v in kern_ms.items()},
                       "folded_kernels": {k: v for k, v in folded.items() if v},
                       "parallelism": f"units sharded over {world} GPU(s), 1 allreduce",
                       "l2": "flushed between timed steps (512 MB write)"},
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3, **e2e_parts},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": frac, "traffic": traffic,
                         "kernel": dom, "kernel_ms_per_step": dom_ms, "kernel_ms_all": kernel_ms,
                         "kernel_launches_per_step": prof.get("launches") if prof else None,
                         "l2_hit_pct": prof.get("l2_hit_pct") if prof else None,
                         "sm_throughput_pct": prof.get("sm_throughput_pct") if prof else None,
                         "l2_throughput_pct": prof.get("l2_throughput_pct") if prof else None,
                         "note": ("frac is the dominant kernel's DRAM traffic over its live time over the "
                                  "measured HBM peak; a low value with a high L2 hit rate means the kernel is "
                                  "not HBM-bound (sm_throughput_pct / l2_throughput_pct, from its ncu --set "
                                  "full capture, say what it is bound by)"),
                         "peak_source": peak_kind,
                         "traffic_source": prof.get("source") if prof else None,
                         "algorithmic": {"value": alg_gbs, "unit": "GB/s",
                                         "frac_of_peak": (alg_gbs / peak) if alg_gbs else None,
                                         "note": "4 B x E / kernel time (E = elements a merge-based level "
                                                 "build consumes); hoisting, probe-side choice and leaf "
                                                 "batching read far fewer bytes, so this exceeds HBM"}},
            "gpu_launches": args.steps * launches_per_step(CONFIG, plans),
            "clocks": clocks.summary(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="BASELINE config (the headline line is cfg2)")
    args = ap.parse_args()
    global CONFIG
    CONFIG = args.config
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
