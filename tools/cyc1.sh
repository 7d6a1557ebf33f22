nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout -k 5 300 python bench.py > gpurun_out/b.log 2>&1; tail -c 600 gpurun_out/b.log
for c in 3 5 4; do timeout -k 5 200 python tools/prof_build.py --config $c --reps 3 2>&1 | tail -3; done
timeout -k 5 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bl_c3.csv python tools/prof_build.py --config 3 --reps 1 > /dev/null 2>&1; python tools/launch_table.py gpurun_out/bl_c3.csv | head -30
