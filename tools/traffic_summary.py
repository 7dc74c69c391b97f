"""DRAM traffic, L2 hit rate and duration per kernel of one bench step, from an
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
lts__t_sector_hit_rate.pct,lts__t_bytes.sum,... --csv` log of
`python tools/ncu_target.py cfgN step 0` (one smg_count_many call; every launch
of a kernel is summed), merged into profiles/ncu_summary.json under
workloads["cfgN:step"].  bench.py reads the dominant kernel's DRAM bytes
(-> roofline.traffic) and L2 hit rate from it.
    python tools/traffic_summary.py OUT.json cfgN:step=LOG.csv [...]"""
import csv
import json
import os
import re
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


def short(name):
    """smg::c4_kernel, count_kernel<0, 0, 1> ... -> c4_kernel, count_kernel"""
    m = re.search(r"(\w+)\s*(<[^(]*>)?\s*\(", name + "(")
    return m.group(1) if m else name


for arg in sys.argv[2:]:
    key, path = arg.split("=", 1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ii, ki, mi, vi = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    launches = {}
    for r in rows[1:]:
        launches.setdefault(r[ii], (short(r[ki]), {}))[1][r[mi]] = float(r[vi].replace(",", ""))
    per = {}
    for _, (k, m) in launches.items():
        p = per.setdefault(k, {"launches": 0, "dram_bytes": 0.0, "duration_ns_under_ncu": 0.0, "l2_bytes": 0.0,
                               "_hit": 0.0})
        p["launches"] += 1
        p["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        p["duration_ns_under_ncu"] += m.get("gpu__time_duration.sum", 0)
        p["l2_bytes"] += m.get("lts__t_bytes.sum", 0)
        p["_hit"] += m.get("lts__t_sector_hit_rate.pct", 0) * m.get("lts__t_bytes.sum", 0)
    for p in per.values():
        p["l2_hit_pct"] = p.pop("_hit") / p["l2_bytes"] if p["l2_bytes"] else None
    doc["workloads"][key] = {
        "source": f"ncu --metrics ... --clock-control none python tools/ncu_target.py {key.replace(':', ' ')} 0 "
                  f"({os.path.basename(path)}); launches of a kernel summed",
        "unit_of_launch": "one bench step (one smg_count_many call over the config's patterns)",
        "per_kernel": per,
    }
json.dump(doc, open(out_path, "w"), indent=1)
print(json.dumps(doc["workloads"], indent=1)[:3000])
