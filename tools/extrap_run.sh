python -m pytest tests/test_gpu.py -x -q -k "shard or validation or golden_corpus or per_root" 2>&1 | tail -5
for cfg in cfg3 cfg4 cfg5; do python -c "from paper_1911_12877_b200 import configs; configs.load('$cfg', verbose=True)"; done
export EXTRAP_BUDGET=150 ORIENT=1
python tools/extrapolate.py cfg4 motif4:star4 32 4096
python tools/extrapolate.py cfg4 motif4:path4 32 4096
python tools/extrapolate.py cfg3 house 32 4096
python tools/extrapolate.py cfg5 pentagon 32 4096
python tools/extrapolate.py cfg5 tailed_diamond_a 32 4096
python tools/extrapolate.py cfg5 tailed_diamond_b 32 4096
