#!/bin/bash
# compute-sanitizer over one small HOT step (the smoke scene, cfg1 stretched): memcheck,
# racecheck (shared-memory hazards: the assembly ring, the smoothers' staging) and synccheck.
# Logs under ${OUT:-gpurun_out/sanitize}.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/$tool.log 2>&1
  echo "rc=$?" >> $OUT/$tool.log
done
