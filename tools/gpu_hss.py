"""HSS diagnostics: keep-count / skeleton mismatches vs goldens."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden, unflatten
import paper_1705_05443_b200 as sg
for name in sys.argv[1:]:
    g = load_golden(name); m = g["meta"]
    X = sg.PointSet(g["X"]); Y = None if g["Y"] is g["X"] else sg.PointSet(g["Y"], role="col")
    tree = sg.build_tree(X, Y, nu0=m["nu0"], mode=m["mode"], tau=m["tau"])
    spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
    M = sg.build_hss(tree, spec, None, None, sg.BuildParams(r=m["r"], tau=m["tau"], eps_svd=m["eps_svd"], basis="interp", rtol=m["rtol"]))
    for side, fac in (("row", M.rowfac), ("col", M.colfac)):
        bad = []
        for i, f in fac.items():
            ref = unflatten(g["skel_%s_ptr" % side], g["skel_%s" % side], i)
            if not np.array_equal(f.skel, ref):
                bad.append((i, f.rank, ref.size))
        print(name, side, "mismatch %d/%d" % (len(bad), len(fac)), bad[:6])
    z = sg.matvec_nodewise(M, g["q"])
    print("  matvec rel %.3e" % (np.linalg.norm(z - g["z"]) / np.linalg.norm(g["z"])))
