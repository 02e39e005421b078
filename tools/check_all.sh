#!/bin/bash
# Timing of the V-cycle / step phases on the bench scenes, then the whole GPU suite.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python tools/vcycle_time.py scenes/cfg2_twisting_bars.json 10 > gpurun_out/vc.log 2>&1
timeout 300 python tools/vcycle_time.py scenes/cfg4_snow.json 5 >> gpurun_out/vc.log 2>&1
timeout 600 python tools/profile_scene.py scenes/cfg2_twisting_bars.json --steps 5 --warmup 2 > gpurun_out/prof.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
