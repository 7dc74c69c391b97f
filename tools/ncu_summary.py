"""Key ncu metrics of a report as markdown + JSON (for profiles/).
    python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX [E_per_launch ...]"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]

rep, prefix = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    rec = {"kernel": r[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            rec[m] = {"value": r[i], "unit": units[i]}
    out.append(rec)
with open(prefix + ".json", "w") as f:
    json.dump(out, f, indent=1)
with open(prefix + ".md", "w") as f:
    f.write(f"# ncu --set full summary: `{rep}`\n\n")
    for rec in out:
        f.write(f"## `{rec['kernel']}`\n\n| metric | value |\n|---|---:|\n")
        for m in METRICS:
            if m in rec:
                f.write(f"| {m} | {rec[m]['value']} {rec[m]['unit']} |\n")
        f.write("\n")
print(open(prefix + ".md").read())
