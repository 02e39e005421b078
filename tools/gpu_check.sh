#!/bin/bash
# Standard GPU-box check: parity tests, smoke, per-phase profile of the bench scene.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:--x} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
HOT_VERBOSE=1 timeout 600 python tools/profile_scene.py ${SCENE:-scenes/cfg2_twisting_bars.json} --steps ${STEPS:-3} --warmup 2 > gpurun_out/prof.log 2>&1; echo prof_rc=$? >> gpurun_out/prof.log
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python tools/profile_scene.py ${SCENE:-scenes/cfg2_twisting_bars.json} --steps 1 --warmup 0 > gpurun_out/ncu_run.log 2>&1
fi
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
fi
