for c in 2 3; do echo cfg $c; timeout -k 5 200 python tools/prof_build.py --config $c --reps 6 2>&1 | tail -3; done
