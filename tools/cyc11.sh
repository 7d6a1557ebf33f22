timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
nproc; timeout -k 5 900 python tools/run_ulv.py 1 4 2>&1 | tail -4
