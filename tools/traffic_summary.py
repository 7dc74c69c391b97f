"""DRAM traffic, L2 hit rate and duration of one count of a pattern from
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
lts__t_sector_hit_rate.pct,... --csv` logs of `tools/ncu_target.py cfg pattern 1`
(the warm-up count and one more; the LAST launch of each kernel is used), merged
into profiles/ncu_summary.json under workloads["cfg:pattern"].  bench.py reads
`dram_bytes_per_launch` (-> roofline.traffic) and `l2_hit_pct` from it.
    python tools/traffic_summary.py OUT.json cfg:pattern=LOG.csv [...]"""
import csv
import json
import os
import sys

out_path = sys.argv[1]
doc = {"workloads": {}}
if os.path.exists(out_path):
    try:
        old = json.load(open(out_path))
        if "workloads" in old:
            doc = old
    except Exception:
        pass
for arg in sys.argv[2:]:
    key, path = arg.split("=", 1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ii, ki, mi, vi = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    launches = {}  # id -> (kernel, {metric: value})
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        launches.setdefault(r[ii], (k, {}))[1][r[mi]] = float(r[vi].replace(",", ""))
    last = {}
    for _, (k, m) in sorted(launches.items(), key=lambda kv: int(kv[0])):
        last[k] = m  # later launches overwrite the warm-up one
    traffic = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in last.values())
    dur = sum(m.get("gpu__time_duration.sum", 0) for m in last.values())
    l2b = sum(m.get("lts__t_bytes.sum", 0) for m in last.values())
    hit = (sum(m.get("lts__t_sector_hit_rate.pct", 0) * m.get("lts__t_bytes.sum", 0) for m in last.values()) / l2b
           if l2b else None)
    doc["workloads"][key] = {
        "source": f"ncu --metrics ... --clock-control none, python tools/ncu_target.py {key.replace(':', ' ')} 1 "
                  f"({os.path.basename(path)})",
        "unit_of_launch": "one count of the pattern (all kernels of the count)",
        "dram_bytes_per_launch": traffic, "duration_ns_under_ncu": dur, "l2_hit_pct": hit,
        "per_kernel": last,
    }
json.dump(doc, open(out_path, "w"), indent=1)
print(json.dumps({k: {x: v[x] for x in ("dram_bytes_per_launch", "duration_ns_under_ncu", "l2_hit_pct")}
                  for k, v in doc["workloads"].items()}, indent=1))
