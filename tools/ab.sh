# A/B timing of library variants on one GPU (used under gpurun):
#   VARIANTS="base _nopipe" CASES="config1 config2 inst:3284 batch:4096" bash tools/ab.sh
# ("base" = the default library _lib/libperseus_b200.so)
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}
mkdir -p gpurun_out
for rep in ${REPS:-1}; do
for v in ${VARIANTS:-base}; do
  [ "$v" = base ] && v=
  echo "#### variant '${v}' rep ${rep}"
  PB_LIB_VARIANT=$v timeout ${CASE_TIMEOUT:-900} python tools/walk_profile.py ${CASES:-config1 config2} 2>&1
done
done
