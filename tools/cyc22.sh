timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log | cut -c1-200
for c in 2 5 1; do timeout -k 5 200 python tools/prof_build.py --config $c --reps 6 2>&1 | tail -3; done
timeout -k 5 300 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -c 3000 gpurun_out/b.log | grep -o '"value": [0-9.]*\|"build_s": [0-9.]*'
