"""Per-launch table (duration, grid, warps active) of an ncu --csv metrics log (tools/compress_levels.sh)."""
import csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
iN, iM, iV, iI = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    d.setdefault(r[iI], {"k": r[iN].split("(")[0][-22:]})[r[iM]] = r[iV].replace(",", "")
for k, v in d.items():
    print("%4s %-24s %10.1f us grid %6s warps %6s" % (k, v["k"], float(v.get("gpu__time_duration.sum", 0)) / 1e3,
          v.get("launch__grid_size"), v.get("sm__warps_active.avg.pct_of_peak_sustained_active")))
