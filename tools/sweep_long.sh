#!/bin/bash
# The long (hub-dominated) BASELINE patterns, one process each, capped.
# usage: tools/sweep_long.sh [cap seconds]
T=${1:-420}
cd "$(dirname "$0")/.."
run() {
  timeout $T python tools/probe_one.py $1 $2 > /tmp/sweep_one.log 2>&1
  rc=$?
  tail -1 /tmp/sweep_one.log
  [ $rc -ne 0 ] && echo "$1 $2: not finished within ${T}s (rc=$rc)"
}
for cfg in cfg4 cfg3 cfg5; do
  python -c "from paper_1911_12877_b200 import configs; configs.load('$cfg', verbose=True)" 2>&1 | tail -1
done
run cfg4 motif4:diamond
run cfg4 motif4:tailed_triangle
run cfg4 motif4:path4
run cfg4 motif4:star4
run cfg3 house
run cfg5 pentagon
run cfg5 tailed_diamond_a
run cfg5 tailed_diamond_b
