mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', d['ms_per_step'], d['e2e']['ms_per_step'])"
python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['counts'])"
python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "bench cfg5 rc=$?"; tail -c 900 gpurun_out/r02_bench_cfg5.json
