"""DRAM traffic of one count (count_kernel + heavy_kernel) from an
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,... --csv` log, as
profiles/ncu_summary.json (bench.py reads `dram_bytes_per_launch` into the
roofline's `traffic`).
    python tools/traffic_summary.py LOG.csv OUT.json "command" """
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = {}
for r in rows[1:]:
    k = r[ki].split("(")[0]
    per.setdefault(k, {})[r[mi]] = float(r[vi].replace(",", ""))
traffic = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
out = {"source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1],
       "unit_of_launch": "one count of the dominant pattern (count_kernel + heavy_kernel)",
       "dram_bytes_per_launch": traffic, "per_kernel": per}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
