# final round-1 validation: GPU tests, smoke, bench (both arms), launch list
timeout -k 5 600 python -m pytest tests/ -m gpu -q > gpurun_out/t_final.log 2>&1; tail -1 gpurun_out/t_final.log
timeout -k 5 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -k 5 400 python bench.py > gpurun_out/bench_final2.log 2>&1; tail -1 gpurun_out/bench_final2.log > gpurun_out/bench_final2.json
timeout -k 5 400 python bench.py --impl reference > gpurun_out/bench_ref2.log 2>&1; tail -1 gpurun_out/bench_ref2.log > gpurun_out/bench_ref2.json
timeout -k 5 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_final2.csv > gpurun_out/launches_final2_summary.txt 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_final2.json')); print({k: d[k] for k in ['value','ms_per_step','build_s','gpu_launches']}, d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
