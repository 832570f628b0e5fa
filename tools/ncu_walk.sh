# ncu evidence for the walk kernels (one GPU; never multi-rank).
#  1. launch list (gpu__time_duration, one pass) of the default bench command
#  2. DRAM traffic + issue metrics of every walk kernel of one launch on the
#     default workload (walk_kernel_wide + walk_kernel; ncu serialises them)
#  3. --set full capture (source page, stall reasons) on a short case
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"walk_kernel" -c 2 --csv --log-file gpurun_out/walk_metrics.csv \
  python tools/walk_profile.py batch:4096 > gpurun_out/ncu_metrics.log 2>&1
if [ -n "$NCU_CASE" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"walk_kernel" -c 1 \
  -o gpurun_out/walk_full python tools/walk_profile.py ${NCU_CASE} > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
fi
