mkdir -p gpurun_out
python -m pytest tests/test_fast.py tests/test_gpu.py -m gpu -q -x -k "k4 or hub or label_free or count_many or motif or cfg2 or shard or adapter" 2>&1 | tail -4
python tools/probe_phases.py cfg2 2 2>&1 | tail -2 | cut -c1-200
python tools/probe_phases.py cfg4 1 2>&1 | tail -1 | cut -c1-250
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_bench_quick.json 2> gpurun_out/r02_bench_quick.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_quick.json')); print(d['ms_per_step'], d['e2e'], d['roofline']['kernel_ms_all'])"
