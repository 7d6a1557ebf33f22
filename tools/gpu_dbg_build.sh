# per-launch warm event timings of the compression launches (SMASH_COMPRESS_DBG) of the last of 2 builds
for c in "$@"; do
  echo "cfg$c"
  SMASH_COMPRESS_DBG=1 python tools/prof_build.py --config $c --reps 2 > gpurun_out/dbg_c$c.log 2>&1
  python - <<PY
import re
L=[l for l in open("gpurun_out/dbg_c$c.log") if l.startswith("compress launch")]
L=L[len(L)//2:]
tot=0
for l in L:
    ms=float(l.rsplit(":",1)[1].split()[0]); tot+=ms
    print(l.strip()[17:])
print("sum %.2f ms"%tot)
print(open("gpurun_out/dbg_c$c.log").read().strip().splitlines()[-1])
PY
done
