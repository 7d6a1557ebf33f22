"""Top source lines by warp-stall samples (and executed warp instructions) from
`ncu -i R --page source --csv --print-source=cuda,sass` (CUDA-line rows only)."""
import csv, sys
path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
key = sys.argv[3] if len(sys.argv) > 3 else "samples"
rows = list(csv.reader(open(path)))
hdr, out, fname = None, [], ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    def num(name):
        try:
            return float(r[hdr.index(name)] or 0)
        except (ValueError, IndexError):
            return 0.0
    s, ins = num("Warp Stall Sampling (All Samples)"), num("Instructions Executed")
    if s > 0 or ins > 0:
        out.append((s, ins, fname, int(r[0]), r[1].strip()[:80]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
idx = 0 if key == "samples" else 1
print("total samples %d  total warp instructions %d" % (ts, ti))
for s, ins, f, ln, src in sorted(out, key=lambda o: -o[idx])[:top]:
    print("%5.1f%% smp %5.1f%% ins  %s:%d  %s" % (100 * s / ts, 100 * ins / ti, f, ln, src))
