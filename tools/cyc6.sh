timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/prof_build.py --config 2 --N 8192 --reps 1 2>&1 | head -40
