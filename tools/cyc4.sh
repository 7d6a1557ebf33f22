timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_compress --launch-skip 4 --launch-count 1 -o gpurun_out/cmp_c2_top -f python tools/prof_build.py --config 2 --reps 1 > gpurun_out/ncu4.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_compress --launch-skip 1 --launch-count 1 -o gpurun_out/cmp_c3_l4 -f python tools/prof_build.py --config 3 --reps 1 > gpurun_out/ncu5.log 2>&1
tail -2 gpurun_out/ncu4.log gpurun_out/ncu5.log
