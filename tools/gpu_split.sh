timeout -k 5 600 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -1
for sp in 0 1; do echo split $sp; for c in 3 5 2; do SMASH_COMPRESS_SPLIT=$sp timeout -k 5 300 python tools/prof_build.py --config $c --reps 4 2>&1 | tail -3 | awk '{print $5}' | tr '\n' ' '; echo; done; done
SMASH_COMPRESS_SPLIT=1 bash tools/compress_levels.sh 3
python tools/level_table.py gpurun_out/cl_c3.csv
