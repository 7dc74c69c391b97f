# Round-2 verification + profile run (one GPU call): parity tests, bench lines, launch list,
# per-kernel traffic of the cfg2 step, one ncu --set full capture per hot kernel.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests.log
tail -4 gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "bench cfg2 rc=$?"
tail -c 1500 gpurun_out/r02_bench_cfg2.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_cfg2_reference.json 2> gpurun_out/r02_bench_cfg2_reference.err; echo "bench ref rc=$?"
python bench.py --config cfg1 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/r02_bench_cfg1.err; echo "bench cfg1 rc=$?"
python bench.py --config cfg4 --steps 2 --warmup 3 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err; echo "bench cfg4 rc=$?"
tail -c 600 gpurun_out/r02_bench_cfg4.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_ncu_launches.log 2>&1; echo "launch list rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k regex:'count_kernel|heavy_kernel|k4_cta_kernel|k4_warp_kernel|c4_kernel|c4_hub_kernel|c4_group_kernel|m4_edge_kernel|m4_edge_counts_kernel|m4_vertex_kernel' --csv \
  --log-file gpurun_out/r02_traffic_cfg2_step.csv python tools/ncu_target.py cfg2 step 0 > gpurun_out/r02_traffic_step.log 2>&1; echo "traffic rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k4_cta_kernel -c 1 -f -o gpurun_out/r02_k4cta_cfg2 \
  python tools/ncu_target.py cfg2 clique4 0 > gpurun_out/r02_ncu_full_k4.log 2>&1; echo "full capture k4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:c4_group_kernel -c 1 -f -o gpurun_out/r02_c4group_cfg2 \
  python tools/ncu_target.py cfg2 rectangle 0 > gpurun_out/r02_ncu_full_c4.log 2>&1; echo "full capture c4 group rc=$?"
python tools/sweep_all.py cfg3 --cap 600 --skip house 2>&1 | grep "^{" | tee gpurun_out/r02_sweep_all_c.log
python tools/motif_fused.py cfg4 2>&1 | tail -1 | tee gpurun_out/r02_motif_fused_cfg4.json
