mkdir -p gpurun_out
python -m pytest tests/test_fast.py tests/test_gpu.py -m gpu -q -x -k "count_many or label_free or motif or adapter or shard" > gpurun_out/r02_gpu_tests_quick.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_gpu_tests_quick.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "bench rc=$?"
tail -c 1200 gpurun_out/r02_bench_cfg2.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_ncu_launches.log 2>&1; echo "launch list rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for pat in rectangle clique4; do
  ncu --metrics $M --clock-control none -k regex:'count_kernel|heavy_kernel|c4_kernel|m4_edge_kernel|m4_vertex_kernel' --csv \
    --log-file gpurun_out/r02_traffic_cfg2_$pat.csv python tools/ncu_target.py cfg2 $pat 1 > gpurun_out/r02_traffic_$pat.log 2>&1; echo "traffic $pat rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:count_kernel -s 1 -c 1 -f -o gpurun_out/r02_count_clique4_cfg2 \
  python tools/ncu_target.py cfg2 clique4 1 > gpurun_out/r02_ncu_full_count.log 2>&1; echo "full capture count rc=$?"
ncu --set full --clock-control none --import-source on -k regex:c4_kernel -s 1 -c 1 -f -o gpurun_out/r02_c4_cfg2 \
  python tools/ncu_target.py cfg2 rectangle 1 > gpurun_out/r02_ncu_full_c4.log 2>&1; echo "full capture c4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:m4_edge_kernel -s 1 -c 1 -f -o gpurun_out/r02_m4edge_cfg2 \
  python tools/ncu_target.py cfg2 rectangle 1 > gpurun_out/r02_ncu_full_edge.log 2>&1; echo "full capture edge rc=$?"
