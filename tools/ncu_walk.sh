# ncu evidence for the walk kernel (one GPU): launch list of a short bench,
# one --set full capture of the walk kernel on a small batch.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --workload batch --batch ${NCU_BATCH:-256} --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 \
  -o gpurun_out/walk_full python tools/walk_profile.py ${NCU_CASE:-config1*1776} > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
