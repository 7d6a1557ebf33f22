# HSS K5 change check: HSS parity (fixtures + full cfg4 census), sharded HSS build, timing, ncu of k_svd
python -m pytest tests/test_fullsize_parity.py -x -q -s -k "4" 2>&1 | grep -E "cfg4|passed|failed|Error|assert" | head -20
python -m pytest tests/test_gpu_parity.py tests/test_ulv.py tests/test_algebra.py tests/test_sharded_build.py -x -q -k "hss or HSS or ulv or cauchy or algebra" 2>&1 | tail -3
SMASH_BUILD_TIMING=1 timeout 300 python tools/prof_build.py --config 4 --reps 2 > gpurun_out/cfg4_levels.txt 2>&1
SMASH_SVD_DBG=1 timeout 300 python tools/prof_build.py --config 4 --reps 1 > gpurun_out/cfg4_svddbg.txt 2>&1
python tools/build_median.py 4 1 --reps 5
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_svd -c 1 -o gpurun_out/svd_l14 -f python tools/prof_build.py --config 4 --reps 1 > gpurun_out/ncu_svd.log 2>&1; echo ncu rc=$?
fi
