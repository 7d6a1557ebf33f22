python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/logtab.log
timeout -k 5 600 python bench.py --no-cpu-baseline > gpurun_out/bench_logtab.log 2>&1; tail -1 gpurun_out/bench_logtab.log > gpurun_out/bench_logtab.json
python -c "
import json; d=json.load(open('gpurun_out/bench_logtab.json')); print({k: d[k] for k in ['value','ms_per_step','build_s']}, d['roofline']['frac'], d['e2e']['value'], d['parity']); print(d['phase_ms_serial']); print({k:(v['build_ms'],v['matvec_ms']) for k,v in d['configs'].items()})" >> gpurun_out/logtab.log 2>&1
cat gpurun_out/logtab.log
