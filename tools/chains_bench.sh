for v in 1 4; do
  echo "== SMASH_QR_CHAINS=$v"
  export SMASH_QR_CHAINS=$v
  for c in 5 2 3; do echo cfg$c; python tools/prof_build.py --config $c --reps 3 2>&1 | tail -1; done
  python -m pytest tests/test_fullsize_parity.py tests/test_gpu_parity.py -q --tb=line -k "skelet or transfer or matvec_vs" 2>&1 | grep -E "passed|failed|factors, [1-9]" | tail -4
done
