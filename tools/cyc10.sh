timeout -k 5 300 python -m pytest tests/test_ulv.py -x -q > gpurun_out/tu.log 2>&1; tail -40 gpurun_out/tu.log
