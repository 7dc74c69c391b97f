#!/bin/bash
# Regenerate the round-2 summaries under profiles/ from the files a GPU call left in gpurun_out/
# (tools/gpu_profile.sh).  Usage: bash tools/make_profiles.sh
set -e
cd "$(dirname "$0")/.."
G=gpurun_out
python tools/summarize_launches.py $G/r02_launches_cfg2.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 1 --no-cpu (cfg2; includes the metering pass: count_kernel<1,...> and heavy_kernel)" > profiles/r02_launches_cfg2.md
rm -f profiles/ncu_summary.json
python tools/traffic_summary.py profiles/ncu_summary.json cfg2:step=$G/r02_traffic_cfg2_step.csv > /dev/null
for r in count_clique4 c4group m4edge; do
  if [ -f $G/r02_${r}_cfg2.ncu-rep ]; then
    cp $G/r02_${r}_cfg2.ncu-rep profiles/
    python tools/ncu_summary.py profiles/r02_${r}_cfg2.ncu-rep profiles/r02_ncu_${r}_cfg2 > /dev/null
  fi
done
cp $G/r02_bench_cfg2.json profiles/r02_bench_cfg2.json
ls -la profiles | grep r02
