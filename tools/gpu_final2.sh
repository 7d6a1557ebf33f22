# final round-2 validation: smoke, bench (both arms), launch list of the bench command
timeout -k 5 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -k 5 600 python bench.py > gpurun_out/bench_r02d.log 2>&1; tail -1 gpurun_out/bench_r02d.log > gpurun_out/bench_r02d.json
timeout -k 5 900 python bench.py --impl reference > gpurun_out/bench_ref_r02d.log 2>&1; tail -1 gpurun_out/bench_ref_r02d.log > gpurun_out/bench_ref_r02d.json
timeout -k 5 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02d.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_r02d.csv > gpurun_out/launches_r02d_summary.txt 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_r02d.json')); print({k: d[k] for k in ['value','ms_per_step','build_s','gpu_launches']}, d['roofline']['frac'], d['roofline']['matvec_total_frac'], d['transfer_roofline']['frac'], d['build_roofline']['frac'], d['e2e']['value'], d['clocks'], d['parity']['pass']); print({k:(round(v['build_ms'],2),round(v['matvec_ms'],3),round(v['matvec_fp64_frac'],3)) for k,v in d['configs'].items()})
r=json.load(open('gpurun_out/bench_ref_r02d.json')); print({k: r.get(k) for k in ['impl','value','ms_per_step','build_s']})"
