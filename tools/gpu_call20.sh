mkdir -p gpurun_out
for i in 1 2; do python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"; done
python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err; echo "bench cfg3 rc=$?"; tail -c 700 gpurun_out/r02_bench_cfg3.json
python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "bench cfg5 rc=$?"; tail -c 700 gpurun_out/r02_bench_cfg5.json
