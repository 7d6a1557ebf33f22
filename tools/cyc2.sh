bash tools/compress_levels.sh 3 2 5
for c in 3 2 5; do python - <<PY
import csv
rows=[r for r in csv.reader(l for l in open("gpurun_out/cl_c$c.csv") if l.startswith('"'))]
h=rows[0]; iN=h.index("Kernel Name"); iM=h.index("Metric Name"); iV=h.index("Metric Value"); iI=h.index("ID")
d={}
for r in rows[1:]:
  d.setdefault(r[iI],{"k":r[iN][:30]})[r[iM]]=r[iV]
print("cfg $c")
for k,v in d.items(): print(k, v)
PY
done
