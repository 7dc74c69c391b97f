python -m pytest tests/test_fast.py -x -q -k "generic_and_oracle" 2>&1 | grep -E "assert|Error|passed|failed" | head -20
