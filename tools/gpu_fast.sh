export SMG_TRACE=1
python -m pytest tests/test_fast.py tests/test_overflow.py tests/test_binding.py tests/test_multirank_gpu.py -x -q 2>&1 | tail -15
for cfg in cfg2 cfg3 cfg4 cfg5; do python -c "from paper_1911_12877_b200 import configs; configs.load('$cfg', verbose=True)"; done
timeout 900 python tools/probe_one.py cfg3 house 2>&1 | grep -v "smg trace\] kernel"
timeout 900 python tools/probe_one.py cfg5 tailed_diamond_b 2>&1 | grep -v "smg trace\] kernel"
timeout 900 python tools/probe_one.py cfg5 tailed_diamond_a 2>&1 | grep -v "smg trace\] kernel"
timeout 400 python tools/probe_one.py cfg4 motif4:path4 2>&1 | grep -v "smg trace\] kernel"
