# ncu launch lists of one warm build per config (2 builds captured, shares per kernel)
for c in 2 3 4 5; do
  python tools/prof_build.py --config $c --reps 2 > gpurun_out/build_t_$c.txt 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/build_launch_$c.csv python tools/prof_build.py --config $c --reps 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/build_launch_$c.csv > gpurun_out/build_table_$c.txt
done
