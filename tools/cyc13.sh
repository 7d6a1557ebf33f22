set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout -k 5 400 python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
timeout -k 5 400 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
timeout -k 5 900 python tools/run_configs.py 1 2 3 4 5 --full-error > gpurun_out/configs_full.jsonl 2> gpurun_out/configs_full.err
timeout -k 5 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
python tools/launch_table.py gpurun_out/launches_final.csv > gpurun_out/launches_final_summary.txt 2>/dev/null
timeout -k 5 600 ncu --set full --import-source on --clock-control none -k regex:k_coupling --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_coupling_final -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout -k 5 600 ncu --set full --import-source on --clock-control none -k regex:k_compress --launch-skip 0 --launch-count 1 -o gpurun_out/ncu_compress_final -f python tools/prof_build.py --config 2 --reps 1 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out | tail -20
