timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for c in 3 5 2 4; do echo cfg $c; timeout -k 5 200 python tools/prof_build.py --config $c --reps 5 2>&1 | tail -3; done
bash tools/compress_levels.sh 3 5 2
for c in 3 5 2; do python tools/level_table.py gpurun_out/cl_c$c.csv 2>/dev/null| head -14; done
