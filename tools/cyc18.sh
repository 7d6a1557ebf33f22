timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log | cut -c1-200
for c in 4 1; do timeout -k 5 300 python tools/prof_build.py --config $c --reps 3 2>&1 | tail -2; done
SMASH_SVD_DBG=1 python tools/prof_build.py --config 4 --reps 1 2>&1 | grep "svd level" | head -2 | cut -c1-250
