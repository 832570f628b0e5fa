# compute-sanitizer runs of the three walk kernels (one GPU); logs -> gpurun_out/
#   memcheck : shared-memory-resident walks (full and partial placement), the
#              global walker, the cooperative kernel (shared and global parents),
#              warm-started get-next chains (the carry buffer)
#   racecheck / synccheck : the cooperative kernel (2 warps, named barriers)
#              and the shared-memory-resident kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS="timeout 900 compute-sanitizer --print-limit 20"
S="gpurun_out/sanitizer.txt"; : > $S
run() { echo "### $*" >> $S; env "$@" >> $S 2>&1; echo "rc=$?" >> $S; }
run PB_SMEM=1 $CS --tool memcheck python tools/walk_profile.py config1 config2
run PB_SMEM=1 PB_SMEM_REGION=6000 $CS --tool memcheck python tools/walk_profile.py config2
run PB_SMEM=0 $CS --tool memcheck python tools/walk_profile.py config2
run $CS --tool memcheck python tools/coop_check.py 2
run PB_WIDE_NO_SHARED_PARENTS=1 $CS --tool memcheck python tools/coop_check.py 2
run $CS --tool racecheck python tools/coop_check.py 2
run $CS --tool synccheck python tools/coop_check.py 2
run $CS --tool memcheck python tools/call_profile.py config1 config2 --calls 20
run $CS --tool racecheck python tools/call_profile.py config1 --calls 10
run PB_SMEM=1 $CS --tool racecheck python tools/walk_profile.py config1
run PB_SMEM=1 $CS --tool synccheck python tools/walk_profile.py config1
grep -E "^###|ERROR SUMMARY|rc=" $S
