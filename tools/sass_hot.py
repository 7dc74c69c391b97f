"""Hot SASS regions of an ncu report (source page, sass view), with stall reasons.
    python tools/sass_hot.py REPORT.ncu-rep [top] [block]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 100
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = [hdr.index(c) for c in cols]
data = [r for r in rows[2:] if len(r) > max(ci)]
tot = sum(int(r[si]) for r in data)
toti = sum(int(r[ii]) for r in data)
st = {c: sum(int(r[i]) for r in data) for c, i in zip(cols, ci)}
T = sum(st.values())
print(f"samples {tot}  warp-instructions {toti:.3e}")
print("stalls:", ", ".join(f"{c[6:]} {100*v/T:.1f}%" for c, v in sorted(st.items(), key=lambda kv: -kv[1]) if v))
regions = {}
for k, r in enumerate(data):
    b = k // blk
    s, n = regions.get(b, (0, 0))
    regions[b] = (s + int(r[si]), n + int(r[ii]))
print(f"\nhottest {blk}-instruction regions: samples%, instr%")
for b, (s, n) in sorted(regions.items(), key=lambda kv: -kv[1][0])[:12]:
    print(f"  [{b*blk:5d}..{b*blk+blk:5d})  {100*s/tot:5.1f}%  {100*n/toti:5.1f}%")
print(f"\ntop {top} instructions:")
for k in sorted(range(len(data)), key=lambda k: -int(data[k][si]))[:top]:
    r = data[k]
    why = max(zip(cols, ci), key=lambda t: int(r[t[1]]))[0][6:]
    print(f"{k:6d} {100*int(r[si])/tot:5.2f}% {100*int(r[ii])/toti:5.2f}%i {why:18s} {r[1].strip()[:60]}")
