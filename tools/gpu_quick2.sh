timeout -k 5 600 python -m pytest tests/ -m gpu -q 2>&1 | tail -1
timeout -k 5 300 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -c 3000 gpurun_out/b.log | grep -o '"value": [0-9.]*\|"build_s": [0-9.]*'
