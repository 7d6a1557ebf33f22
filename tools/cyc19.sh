timeout -k 5 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:k_ulv --csv --log-file gpurun_out/ulv4.csv python tools/prof_ulv.py --config 4 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ulv4.csv
python tools/level_table.py gpurun_out/ulv4.csv | awk '{print $2, $(NF-5), $(NF-2)}' | sort -k2 -g -r | head -12
