# matvec-only check: parity tests of the matvec + cfg5 / cfg3 / cfg2 timings
python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py tests/test_fullsize_parity.py -q -x -k "matvec or block or dense or kernel" 2>&1 | tail -2 > gpurun_out/mv_quick.log
for c in 5 3 2 1; do python tools/run_configs.py $c 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/mv_quick.log; done
cat gpurun_out/mv_quick.log
