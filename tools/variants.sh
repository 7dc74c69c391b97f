#!/bin/bash
# Time prebuilt engine variants (exp_variants/*.so, tuning builds) on cfg2:
# each is copied over the in-tree engine for its run; the default is restored.
cd "$(dirname "$0")/.."
cp paper_1911_12877_b200/libsymmine_gpu.so /tmp/engine_default.so
for v in "$@"; do
  cp exp_variants/$v.so paper_1911_12877_b200/libsymmine_gpu.so
  echo "== $v"
  for label in rectangle clique4; do timeout 300 python tools/probe_one.py cfg2 $label 2>&1 | tail -1; done
done
cp /tmp/engine_default.so paper_1911_12877_b200/libsymmine_gpu.so
