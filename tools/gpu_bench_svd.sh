# bench line (cfg5 headline + configs 1-4) and an ncu capture of the cfg4 leaf-level k_svd launches
timeout -k 5 600 python bench.py > gpurun_out/bench_r02c.log 2>&1; tail -1 gpurun_out/bench_r02c.log > gpurun_out/bench_r02c.json
python -c "
import json; d=json.load(open('gpurun_out/bench_r02c.json')); print({k: d[k] for k in ['value','ms_per_step','build_s']}, d['roofline']['frac'], d['e2e']['value']); print({k:(v['build_ms'],v['matvec_ms']) for k,v in d['configs'].items()})"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_svd -c 2 -o gpurun_out/svd_split_r02 -f python tools/prof_build.py --config 4 --reps 1 > gpurun_out/ncu_svd2.log 2>&1; tail -2 gpurun_out/ncu_svd2.log
