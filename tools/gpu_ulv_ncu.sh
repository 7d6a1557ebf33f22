# ncu --set full of the leaf-level ULV kernels (cfg4): factor reduce, solve up, solve down
timeout -k 5 600 ncu --set full --clock-control none -k regex:k_ulv_reduce --launch-skip 0 --launch-count 1 -o gpurun_out/ulvf_red -f python tools/prof_ulv.py --config 4 > /dev/null 2>&1
timeout -k 5 600 ncu --set full --clock-control none -k regex:k_ulv_up --launch-skip 0 --launch-count 1 -o gpurun_out/ulvf_up -f python tools/prof_ulv.py --config 4 > /dev/null 2>&1
timeout -k 5 600 ncu --set full --clock-control none -k regex:k_ulv_down --launch-skip 12 --launch-count 1 -o gpurun_out/ulvf_down -f python tools/prof_ulv.py --config 4 > /dev/null 2>&1
echo ok
