python -m pytest tests/test_fast.py -x -q 2>&1 | tail -5
for cfg in cfg4 cfg5; do python -c "from paper_1911_12877_b200 import configs; configs.load('$cfg', verbose=True)"; done
timeout 900 python tools/probe_one.py cfg4 motif4:star4
timeout 1500 python tools/probe_one.py cfg5 tailed_diamond_a
