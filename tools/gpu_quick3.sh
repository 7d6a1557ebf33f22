timeout -k 5 600 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -2
for c in 2 5 3; do timeout -k 5 200 python tools/prof_build.py --config $c --reps 5 2>&1 | tail -2; done
timeout -k 5 300 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -c 3000 gpurun_out/b.log | grep -o '"value": [0-9.]*\|"build_s": [0-9.]*'
