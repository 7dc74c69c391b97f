#!/bin/bash
# Timing experiments on one config: tools/exp.sh cfgN "label ..." "ENV=val ..." ...
# Each env setting (a quoted word; "-" = defaults) runs every label once.
cd "$(dirname "$0")/.."
cfg=$1; labels=$2; shift 2
python -c "from paper_1911_12877_b200 import configs; configs.load('$cfg', verbose=True)" 2>&1 | tail -1
for envs in "$@"; do
  [ "$envs" = "-" ] && envs=""
  for label in $labels; do
    echo "== $envs $label"
    env $envs timeout 300 python tools/probe_one.py $cfg $label 2>&1 | tail -2
  done
done
