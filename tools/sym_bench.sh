python -m pytest tests/test_coupling_sym.py -q -x --tb=short 2>&1 | tail -3
for v in 0 1; do
  echo "== SMASH_COUPLING_SYM=$v"
  for c in 5 2; do SMASH_COUPLING_SYM=$v python bench.py --config $c --steps 10 --warmup 3 --no-extras --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_serial']; print('cfg', d['config']['config_id'], 'matvec %.3f coupling %.3f near %.3f parity %s' % (d['ms_per_step'], p['coupling'], p['nearfield'], d['parity'] and d['parity'].get('pass')))"; done
done
