timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for c in 2 5 3; do timeout -k 5 200 python tools/prof_build.py --config $c --reps 6 2>&1 | tail -3; done
