mkdir -p gpurun_out
python -m pytest tests/test_fast.py -m gpu -q -x -k "hub or label_free or count_many" 2>&1 | tail -3
for gd in 0 512 128 2048; do
  echo "== SMG_M4_GROUP_DEGREE=$gd"
  SMG_M4_GROUP_DEGREE=$gd python tools/probe_phases.py cfg2 2 2>&1 | tail -2 | cut -c1-120
  SMG_M4_GROUP_DEGREE=$gd python tools/probe_phases.py cfg4 1 2>&1 | tail -1 | cut -c1-120
done 2>&1 | tee gpurun_out/r02_group_threshold.log
