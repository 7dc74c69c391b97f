# round-2 GPU call 1: parity tests, cfg2 bench, pentagon extrapolations
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests.log
tail -5 gpurun_out/r02_gpu_tests.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench_cfg2.json
python -c "from paper_1911_12877_b200 import configs; configs.load('cfg5', verbose=True)"
export EXTRAP_BUDGET=120
for o in "" asc desc; do ORIENT=$o timeout 600 python tools/extrapolate.py cfg5 pentagon 24 4096 2>&1 | tail -2 | tee -a gpurun_out/r02_extrap_pentagon.log; done
