# HSS round trip: census tests (fixtures + full cfg4), cfg4 build time, optional per-level SVD trace
python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -s --tb=short -k "(skeletons or transfer or matvec or hss) and (hss or cfg4 or cfg1 or 4)" 2>&1 | grep -E "factors|passed|failed|exact|Error|assert" | cut -c1-300 > gpurun_out/hss_cycle.log
python tools/prof_build.py --config 4 --reps 4 2>&1 | tail -3 >> gpurun_out/hss_cycle.log
SMASH_SVD_DBG=1 SMASH_BUILD_TIMING=1 timeout 300 python tools/prof_build.py --config 4 --reps 2 > gpurun_out/svd_dbg_c4.log 2>&1
grep "^level" gpurun_out/svd_dbg_c4.log | tail -26 | awk '{print $2, $4, $11}' | tr '\n' ';' >> gpurun_out/hss_cycle.log
cat gpurun_out/hss_cycle.log
