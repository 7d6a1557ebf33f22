timeout -k 5 300 python -m pytest tests/test_container.py -x -q > gpurun_out/tc.log 2>&1; tail -30 gpurun_out/tc.log
