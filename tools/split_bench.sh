for v in 1 0; do
  echo "== NOSPLIT=$v"
  for c in 5 3 2 4 1; do if [ $v = 1 ]; then export SMASH_COMPRESS_NOSPLIT=1; else unset SMASH_COMPRESS_NOSPLIT; fi; echo cfg$c; python tools/prof_build.py --config $c --reps 3 2>&1 | tail -2; done
done
unset SMASH_COMPRESS_NOSPLIT
python -m pytest tests/test_fullsize_parity.py tests/test_gpu_parity.py -q -x --tb=short -k "skelet or transfer" 2>&1 | tail -3
