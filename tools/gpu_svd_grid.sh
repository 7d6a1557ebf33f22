for k in 2 4 2 4; do echo "per_sm $k: $(SMASH_SVD_PER_SM=$k SMASH_BUILD_TIMING=1 timeout -k 5 300 python tools/prof_build.py --config 4 --reps 3 2>&1 | grep 'level 14 side 0' | tail -1)"; done
