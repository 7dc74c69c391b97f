mkdir -p gpurun_out
python -m pytest tests/test_fast.py -m gpu -q -x -k "hub or label_free or count_many" 2>&1 | tail -3
for hd in 16384 4096 1024 256; do
  echo "== SMG_M4_HUB_DEGREE=$hd"
  SMG_M4_HUB_DEGREE=$hd SMG_TRACE=1 python tools/probe_one.py cfg2 rectangle 2>&1 | grep -E "m4 sums|cfg2 rect" | sed 's/C4=.*STAR=0//' 
  SMG_M4_HUB_DEGREE=$hd SMG_TRACE=1 python tools/probe_one.py cfg4 motif4:rectangle 2>&1 | grep -E "m4 sums|cfg4 motif" | sed 's/C4=.*STAR=0//'
done 2>&1 | tee gpurun_out/r02_hub_threshold.log
