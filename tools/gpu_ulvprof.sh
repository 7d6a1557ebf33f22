timeout -k 5 600 ncu --set full --import-source on --clock-control none -k regex:k_ulv_down --launch-skip 12 --launch-count 1 -o gpurun_out/ulv_down -f python tools/prof_ulv.py --config 4 > gpurun_out/ulvprof.log 2>&1
timeout -k 5 600 ncu --set full --import-source on --clock-control none -k regex:k_ulv_up --launch-skip 0 --launch-count 1 -o gpurun_out/ulv_up -f python tools/prof_ulv.py --config 4 > gpurun_out/ulvprof2.log 2>&1
tail -2 gpurun_out/ulvprof.log
