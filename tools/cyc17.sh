timeout -k 5 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/c4.csv python tools/prof_build.py --config 4 --reps 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/c4.csv 2>/dev/null | head -12
python tools/level_table.py gpurun_out/c4.csv | sort -k4 -n -r -t' ' | head -5
