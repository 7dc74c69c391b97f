#!/bin/bash
# Time every BASELINE pattern on its config (one process per pattern, bounded).
# usage: tools/sweep.sh [per-pattern timeout s] [cfg ...]
T=${1:-300}; shift
CFGS=${@:-cfg1 cfg2 cfg3 cfg4 cfg5}
cd "$(dirname "$0")/.."
for cfg in $CFGS; do
  python -c "from paper_1911_12877_b200 import configs; configs.load('$cfg', verbose=True)" 2>&1 | tail -1
  for label in $(python -c "from paper_1911_12877_b200 import configs; print(' '.join(l for l,_ in configs.config_patterns('$cfg')))"); do
    timeout $T python tools/probe_one.py $cfg $label > /tmp/sweep_one.log 2>&1
    rc=$?
    tail -1 /tmp/sweep_one.log
    [ $rc -ne 0 ] && echo "$cfg $label: not finished within ${T}s (rc=$rc)"
  done
done
