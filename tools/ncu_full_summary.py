"""Key metrics of every kernel in an `ncu --set full` report (the profiles/*_ncu_full_summary.txt
format).  Usage: python tools/ncu_full_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sectors_srcunit_tex_op_read.sum", "dram__bytes_read.sum.per_second",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
idx = {k: i for i, k in enumerate(hdr)}
for r in rows[2:]:
    print(f"kernel: {r[idx['Kernel Name']].split('(')[0]}")
    for k in KEYS:
        if k in idx:
            print(f"  {k} = {r[idx[k]]} {units[idx[k]]}")
    print()
