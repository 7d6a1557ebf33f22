"""Per-level factor statistics (count, |ibar|, rank) of a built config (GPU)."""
import argparse, collections, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--N", type=int, default=None)
a = ap.parse_args()
c = CONFIGS[a.config]
X, Y, rng = make_points(a.config, N=a.N)
spec, params = build_params(a.config)
tree = sg.build_tree(sg.PointSet(X), None if Y is X else sg.PointSet(Y), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
M = (sg.build_h2 if c["structure"] == "h2" else sg.build_hss)(tree, spec, None, None, params)
A = tree.arrays()
E = M.export_side(0)
nib = np.diff(E["perm_ptr"])
st = collections.defaultdict(list)
for i in np.nonzero(E["has"])[0]:
    st[int(A["level"][i])].append((int(nib[i]), int(E["rank"][i]), A["child_ptr"][i + 1] == A["child_ptr"][i]))
for l in sorted(st):
    v = np.array(st[l])
    print("level %2d nodes %6d leaves %6d nib mean %6.1f max %4d rank mean %5.1f max %3d  full-rank %d"
          % (l, len(v), v[:, 2].sum(), v[:, 0].mean(), v[:, 0].max(), v[:, 1].mean(), v[:, 1].max(),
             (v[:, 0] == v[:, 1]).sum()))
print("pairs L", len(M.pairs_L), "Lm", len(M.pairs_Lm))
