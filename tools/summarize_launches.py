"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and mean device time, share of the total.
    python tools/summarize_launches.py gpurun_out/launches.csv > profiles/rNN_launches.md"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = OrderedDict()
seq = []
for r in rows[1:]:
    name = r[ki].split("(")[0] if "<" not in r[ki] else r[ki].split(">(")[0] + ">"
    t = float(r[vi].replace(",", ""))
    agg.setdefault(name, []).append(t)
    seq.append((name, t))
total = sum(t for _, t in seq)
print(f"# ncu launch list: `{' '.join(sys.argv[2:]) or 'see header'}`\n")
print("gpu__time_duration.sum per launch, --clock-control none (cold caches, serialised).\n")
print("| kernel | launches | total ms | mean ms | share |")
print("|---|---:|---:|---:|---:|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"| `{k}` | {len(v)} | {sum(v)/1e6:.3f} | {sum(v)/len(v)/1e6:.3f} | {100*sum(v)/total:.1f}% |")
print(f"\nTotal device time: {total/1e6:.1f} ms over {len(seq)} launches.\n")
print("## Launch sequence\n")
print("| # | kernel | ms |")
print("|---:|---|---:|")
for i, (k, t) in enumerate(seq):
    print(f"| {i} | `{k}` | {t/1e6:.3f} |")
