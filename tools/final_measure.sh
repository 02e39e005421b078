#!/bin/bash
# Round measurement set (one GPU): smoke, bench (ours + the reference arm on the full scene), the
# ncu launch list of the bench command, per-kernel DRAM bytes of one headline step, and one ncu
# --set full capture of the dominant kernels.  Outputs under gpurun_out/${TAG:-final}; summaries
# are copied into profiles/ by hand.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/${TAG:-final}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo bench_rc=$? >> $O/bench.log
if [ -z "$NO_REF" ]; then
  timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo ref_rc=$? >> $O/bench_ref.log
fi
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs"
timeout 600 $CMD > $O/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo launch_rc=$? >> $O/ncu_launch.log
PCMD="python tools/profile_scene.py scenes/cfg2_twisting_bars.json --steps 1 --warmup 2"
timeout 300 $PCMD > $O/prof_short.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/dram.csv $PCMD > $O/ncu_dram.log 2>&1
echo dram_rc=$? >> $O/ncu_dram.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_bin_pairs|k_row_gather|k_sgs_stream|k_sgs_flow|k_bin_p2g|k_bin_force" \
  -c 10 -f -o $O/full $PCMD > $O/ncu_full.log 2>&1
echo full_rc=$? >> $O/ncu_full.log
