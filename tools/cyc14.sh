for cfg in "0 32" "64 32" "64 64" "128 64" "40 32"; do set -- $cfg; echo "tiny $1 threads $2"; for c in 2 5 3; do SMASH_COMPRESS_TINY=$1 SMASH_COMPRESS_TINY_T=$2 timeout -k 5 200 python tools/prof_build.py --config $c --reps 5 2>&1 | tail -2 | head -1; done; done
SMASH_COMPRESS_TINY=64 SMASH_COMPRESS_TINY_T=32 bash tools/compress_levels.sh 2 5
for c in 2 5; do python tools/level_table.py gpurun_out/cl_c$c.csv | head -8; done
SMASH_COMPRESS_TINY=64 SMASH_COMPRESS_TINY_T=32 timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
