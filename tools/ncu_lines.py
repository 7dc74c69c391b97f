"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo).
    python tools/ncu_lines.py REPORT [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
lines = []
for r in rows:
    if r and r[0].isdigit() and len(r) > si and r[si].isdigit():
        lines.append((int(r[si]), int(r[0]), r[1][:90], r[ii]))
tot = sum(x[0] for x in lines)
print(f"total samples {tot}")
for s, ln, src, ie in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% line {ln:5d} inst={ie:>12}  {src}")
