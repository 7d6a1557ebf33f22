"""Print the per-level compression launches captured by tools/compress_levels.sh."""
import csv, sys
for c in sys.argv[1:]:
    lines = [l for l in open("gpurun_out/cl_c%s.csv" % c) if l.startswith('"')]
    rows = list(csv.reader(lines)); h = rows[0]
    iid, im, iv, ik = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Kernel Name")
    d = {}
    for r in rows[1:]:
        d.setdefault(r[iid], {"name": r[ik].split("(")[0][-40:]})[r[im]] = r[iv]
    tot = 0.0
    print("cfg", c)
    for k, v in d.items():
        us = float(v["gpu__time_duration.sum"].replace(",", "")) / 1000
        tot += us
        print("  %-40s grid %6s block %5s cl %s %10.1f us warps %s" % (
            v["name"], v.get("launch__grid_size"), v.get("launch__block_size"), v.get("launch__cluster_dim_x"),
            us, v.get("sm__warps_active.avg.pct_of_peak_sustained_active")))
    print("  total %.1f us" % tot)
