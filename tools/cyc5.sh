timeout -k 5 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
export SMASH_LIB=$PWD/paper_1705_05443_b200/libsmash_b200_trace.so
for c in 2 3 5; do echo cfg $c; timeout -k 5 200 python tools/prof_build.py --config $c --reps 1 2>&1 | grep -v "^tree" | tail -14; done
unset SMASH_LIB
for c in 2 3 5 1; do echo cfg $c; timeout -k 5 200 python tools/prof_build.py --config $c --reps 3 2>&1 | tail -2; done
