# transfer-pass G staging chunk sweep (SMASH_XFER_GKB): isolated phase times per config
for kb in 64 32 16 8; do
  for c in 5 2 3; do
    echo "== GKB $kb cfg $c" >> gpurun_out/xfer_sweep.log
    SMASH_XFER_GKB=$kb python bench.py --config $c --steps 5 --warmup 2 --no-extras --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_serial']; print('matvec %.3f up %.3f down %.3f leaf %.3f frac %.3f' % (d['ms_per_step'], p['upward'], p['downward'], p['leaf_farfield'], d['transfer_roofline']['frac']))" >> gpurun_out/xfer_sweep.log
  done
done
