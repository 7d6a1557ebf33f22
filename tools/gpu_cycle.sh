timeout -k 5 400 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
SMASH_MATVEC_SERIAL=1 timeout -k 5 200 python bench.py --no-cpu-baseline > gpurun_out/bs.log 2>&1; tail -c 1500 gpurun_out/bs.log | grep -o "phase_ms[^}]*"
timeout -k 5 200 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -c 2500 gpurun_out/b.log | grep -o "\"value\": [0-9.]*\|phase_ms[^}]*"
timeout -k 5 100 python tools/prof_matvec.py --reps 3 > /dev/null && timeout -k 5 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mv_launch.csv python tools/prof_matvec.py --reps 3 > /dev/null 2>&1
