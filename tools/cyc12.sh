timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for nw in 0 128; do echo narrow $nw; for c in 2 5 3; do SMASH_COMPRESS_NARROW=$nw timeout -k 5 200 python tools/prof_build.py --config $c --reps 5 2>&1 | tail -2; done; done
bash tools/compress_levels.sh 2
python tools/level_table.py gpurun_out/cl_c2.csv
