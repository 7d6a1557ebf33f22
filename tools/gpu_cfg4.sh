# HSS cfg4 build: per-level host timing (SMASH_BUILD_TIMING) and end-to-end build times
SMASH_BUILD_TIMING=1 timeout -k 5 300 python tools/prof_build.py --config 4 --reps 4 > /tmp/o.txt 2>&1
grep "^tree" /tmp/o.txt | awk '{print $5}' | tr '\n' ' '; echo; grep "level 14 side 0\|level 13 side 0" /tmp/o.txt | tail -2
