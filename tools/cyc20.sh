timeout -k 5 300 python -m pytest tests/test_ulv.py tests/test_container.py -x -q 2>&1 | tail -2
timeout -k 5 300 python tools/run_ulv.py 1 4 --reps 5 > gpurun_out/ulv.jsonl 2>&1; cat gpurun_out/ulv.jsonl | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print(d['cfg'], d['ulv_factor_ms'], d['ulv_solve_ms_min'], d['residual_rel'], d['gpu_vs_oracle_x_rel'])"
