# full GPU suite + cfg4 build timing (default and internal floor 2^-57)
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_full.log
python tools/prof_build.py --config 4 --reps 5 2>&1 | tail -4 >> gpurun_out/gpu_full.log
echo "floor 57" >> gpurun_out/gpu_full.log
SMASH_SVD_FLOOR=57 python tools/prof_build.py --config 4 --reps 5 2>&1 | tail -4 >> gpurun_out/gpu_full.log
SMASH_SVD_FLOOR=57 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -s --tb=short -k "(skeletons or transfer or matvec or hss) and (hss or cfg4 or cfg1 or 4)" 2>&1 | grep -E "factors|passed|failed|exact" | cut -c1-200 >> gpurun_out/gpu_full.log
cat gpurun_out/gpu_full.log
