# GPU check used during development: parity tests, per-phase profile, short bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 600 python tools/walk_profile.py ${PROFILE_CASES:-config1 config2 config3 config4 batch:256} 2>&1 | tee gpurun_out/walk_profile.log
if [ -n "$BENCH_ARGS" ]; then timeout 900 python bench.py $BENCH_ARGS 2>&1 | tail -3 | tee gpurun_out/bench.log; fi
