timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for c in 2 3 5 1; do echo cfg $c; timeout -k 5 200 python tools/prof_build.py --config $c --reps 3 2>&1 | tail -2; done
echo gper4; SMASH_GWS_PER_SM=4 timeout -k 5 200 python tools/prof_build.py --config 3 --reps 3 2>&1 | tail -2
bash tools/compress_levels.sh 3 5 2
for c in 3 5 2; do python tools/level_table.py gpurun_out/cl_c$c.csv 2>/dev/null| head -14; done
