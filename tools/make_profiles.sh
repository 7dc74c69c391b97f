#!/bin/bash
# Regenerate the round-2 summaries under profiles/ from the files a GPU call left in gpurun_out/
# (tools/gpu_profile.sh).  Usage: bash tools/make_profiles.sh
set -e
cd "$(dirname "$0")/.."
G=gpurun_out
python tools/summarize_launches.py $G/r02_launches_cfg2.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 1 --no-cpu (cfg2; includes the metering pass: count_kernel<1,...> and heavy_kernel)" > profiles/r02_launches_cfg2.md
rm -f profiles/ncu_summary.json
python tools/traffic_summary.py profiles/ncu_summary.json cfg2:step=$G/r02_traffic_cfg2_step.csv > /dev/null
for r in k4cta c4group m4edge; do
  if [ -f $G/r02_${r}_cfg2.ncu-rep ]; then
    cp $G/r02_${r}_cfg2.ncu-rep profiles/
    python tools/ncu_summary.py profiles/r02_${r}_cfg2.ncu-rep profiles/r02_ncu_${r}_cfg2 > /dev/null
  fi
done
cp $G/r02_bench_cfg2.json profiles/r02_bench_cfg2.json
ls -la profiles | grep r02
# merge the --set full utilisation figures into ncu_summary.json (bench.py copies them into the roofline object)
python - <<'PY'
import json
doc = json.load(open("profiles/ncu_summary.json"))
per = doc["workloads"]["cfg2:step"]["per_kernel"]
for kernel, rep in (("k4_cta_kernel", "k4cta"), ("c4_group_kernel", "c4group"), ("m4_edge_kernel", "m4edge")):
    try:
        rec = json.load(open(f"profiles/r02_ncu_{rep}_cfg2.json"))[0]
    except Exception:
        continue
    if kernel in per:
        for key, name in (("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
                          ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_throughput_pct"),
                          ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
                          ("launch__registers_per_thread", "registers_per_thread")):
            if key in rec:
                per[kernel][name] = float(rec[key]["value"])
        per[kernel]["full_capture"] = f"profiles/r02_{rep}_cfg2.ncu-rep"
json.dump(doc, open("profiles/ncu_summary.json", "w"), indent=1)
PY
