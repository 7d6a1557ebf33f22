for nw in 128 160 256; do echo narrow $nw; for c in 2 5; do SMASH_COMPRESS_NARROW=$nw timeout -k 5 200 python tools/prof_build.py --config $c --reps 6 2>&1 | tail -3 | sort | head -1; done; done
SMASH_COMPRESS_NARROW=160 bash tools/compress_levels.sh 2
python tools/level_table.py gpurun_out/cl_c2.csv
