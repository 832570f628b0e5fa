cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/walk_c1 python tools/walk_profile.py config1 > gpurun_out/ncu_c1.log 2>&1
tail -3 gpurun_out/ncu_c1.log
