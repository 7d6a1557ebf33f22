# warm build times per config (tree + compression), 3 reps each
for c in 1 2 3 4 5; do echo "cfg$c"; python tools/prof_build.py --config $c --reps 3 2>&1 | tail -2; done
