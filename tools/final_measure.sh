#!/bin/bash
# Round-end measurement set (one GPU): parity suite + smoke, bench (ours + reference arm), the ncu
# launch list of the bench command, one ncu --set full capture of the dominant kernels, and the
# one-GPU slab emulation.  Outputs under gpurun_out/; summaries are copied into profiles/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$? >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$? >> gpurun_out/ncu_launch.log
PCMD="python tools/profile_scene.py scenes/cfg2_twisting_bars.json --steps 1 --warmup 0"
timeout 300 $PCMD > gpurun_out/prof_short.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_assemble_rows|k_sgs_stream" -c 2 -f -o gpurun_out/full $PCMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$? >> gpurun_out/ncu_full.log
timeout 900 python tools/slab_emulate.py --ranks 1,2,4,8 --steps 8 --warmup 4 --repeat 2 > gpurun_out/emulate.log 2>&1; echo rc=$? >> gpurun_out/emulate.log
