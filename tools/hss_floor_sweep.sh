# HSS SVD truncation sweep: skeleton census (fixtures + full cfg4) and cfg4 build time per floor
# FLOORS="internal:leaf ..." (SMASH_SVD_FLOOR / SMASH_SVD_FLOOR_LEAF)
for p in ${FLOORS:-58:58}; do
  e=${p%%:*}; lf=${p##*:}
  echo "== floor 2^-$e leaves 2^-$lf" >> gpurun_out/hss_sweep2.log
  SMASH_SVD_FLOOR=$e SMASH_SVD_FLOOR_LEAF=$lf python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py -q -s --tb=no -k "(skeletons or transfer or matvec) and (hss or cfg4 or cfg1 or 4)" 2>&1 | grep -E "factors|passed|failed|exact" >> gpurun_out/hss_sweep2.log
  SMASH_SVD_FLOOR=$e SMASH_SVD_FLOOR_LEAF=$lf python tools/prof_build.py --config 4 --reps 3 2>&1 | tail -1 >> gpurun_out/hss_sweep2.log
done
