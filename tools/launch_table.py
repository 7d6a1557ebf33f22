"""Summarise an ncu --csv launch list: the kernels after the last occurrence of
a marker kernel (one matvec), or totals by kernel name."""
import csv, sys, collections
path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else None
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
i_n, i_v = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[i_n], float(r[i_v].replace(",", "")) / 1000) for r in rows[1:] if len(r) > i_v]
if marker:
    idx = [i for i, (n, _) in enumerate(ks) if marker in n]
    sel = ks[idx[-1]:]
    for n, v in sel:
        print("%-70s %9.1f us" % (n[:70], v))
    print("total %.1f us" % sum(v for _, v in sel))
else:
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in ks:
        a = agg[n.split("(")[0][:70]]
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-70s launches %5d total %10.1f us avg %8.2f us share %5.1f%%" % (n, c, v, v / c, 100 * v / tot))
