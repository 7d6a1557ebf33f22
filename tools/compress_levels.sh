#!/bin/bash
# ncu launch list of the compression kernels of one build per config (grid, block, duration)
for c in "$@"; do
  timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:"k_compress|k_svd" --log-file gpurun_out/cl_c$c.csv python tools/prof_build.py --config $c --reps 1 > gpurun_out/cl_c$c.log 2>&1
done
