# reference arm on the default (cfg5) workload + a launch list of the bench
( time python bench.py --impl reference --steps 10 --warmup 3 ) > gpurun_out/ref_cfg5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/launch_table.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5_summary.txt
tail -2 gpurun_out/ref_cfg5.log
