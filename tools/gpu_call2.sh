# round-2 GPU call 2: parity tests, cfg2 bench, launch list, traffic, full ncu capture, pentagon estimate
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests.log
tail -5 gpurun_out/r02_gpu_tests.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02_bench_cfg2.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_ncu_launches.log 2>&1; echo "launch list rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for pat in rectangle clique4; do
  ncu --metrics $M --clock-control none -k regex:'rect_kernel|count_kernel|heavy_kernel' --csv \
    --log-file gpurun_out/r02_traffic_cfg2_$pat.csv python tools/ncu_target.py cfg2 $pat 1 > gpurun_out/r02_traffic_$pat.log 2>&1; echo "traffic $pat rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:rect_kernel -c 1 -f -o gpurun_out/r02_rect_cfg2 \
  python tools/ncu_target.py cfg2 rectangle 0 > gpurun_out/r02_ncu_full.log 2>&1; echo "full capture rc=$?"
EXTRAP_BUDGET=500 timeout 900 python tools/extrap_strat.py cfg5 pentagon 2 65536 2>&1 | tail -12 | tee gpurun_out/r02_extrap_pentagon_asc.log
