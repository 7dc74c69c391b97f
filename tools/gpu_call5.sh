mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests.log
tail -5 gpurun_out/r02_gpu_tests.log
SMG_TRACE=1 python tools/probe_one.py cfg2 rectangle 2>&1 | grep -v "kernel [0-9.]* ms:" | tail -5
python tools/sweep_all.py cfg1 cfg2 cfg4 --cap 600 2>&1 | grep "^{" | tee gpurun_out/r02_sweep_all_b.log
python tools/motif_fused.py cfg4 2>&1 | tail -1 | tee gpurun_out/r02_motif_fused_cfg4.json
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/r02_bench_cfg2.json
