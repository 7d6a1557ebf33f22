for e in 53 55 56 58 60 63; do
  echo "== floor 2^-$e" >> gpurun_out/hss2.log
  SMASH_SVD_FLOOR=$e python -m pytest tests/test_fullsize_parity.py -q -s --tb=no -k "skeletons and 4" 2>&1 | grep factors >> gpurun_out/hss2.log
  SMASH_SVD_FLOOR=$e python bench.py --config 4 --steps 5 --warmup 2 --no-extras --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('build_s', d['build_s'], 'err', d['parity']['err_vs_exact'])" >> gpurun_out/hss2.log 2>&1
done
