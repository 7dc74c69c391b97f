mkdir -p gpurun_out
python -m pytest tests/test_fast.py tests/test_gpu.py -m gpu -q -x -k "k4 or hub or label_free or count_many or motif or cfg2 or shard" 2>&1 | tail -5
python tools/probe_phases.py cfg2 2 2>&1 | tail -2 | cut -c1-200
python tools/probe_phases.py cfg4 1 2>&1 | tail -1 | cut -c1-200
python tools/sweep_all.py cfg2 cfg3 --cap 300 --skip house rectangle 2>&1 | grep "^{" | cut -c1-200
SMG_K4=0 python tools/probe_phases.py cfg2 1 2>&1 | tail -1 | cut -c1-200
