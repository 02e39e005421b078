timeout 200 python tools/asm_cmp.py scenes/cfg1_cube.json 3 2000 2>&1 | tail -1
timeout 500 python tools/asm_cmp.py scenes/cfg2_twisting_bars.json 5 60000 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bin_pairs|k_row_gather" -c 2 python tools/asm_ab.py scenes/cfg2_twisting_bars.json 1 2>&1 | grep -E "k_bin_pairs|k_row_gather|duration|dram__|tensor"
