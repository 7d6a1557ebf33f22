"""Quick GPU sanity run: build + matvec on a golden case, print diagnostics."""
import sys, time
import numpy as np
sys.path.insert(0, "tests")
from conftest import load_golden, unflatten
import paper_1705_05443_b200 as sg
for name in sys.argv[1:]:
    g = load_golden(name)
    m = g["meta"]
    X = sg.PointSet(g["X"])
    Y = None if g["Y"] is g["X"] else sg.PointSet(g["Y"], role="col")
    t0 = time.time()
    tree = sg.build_tree(X, Y, nu0=m["nu0"], mode=m["mode"], tau=m["tau"])
    A = tree.arrays()
    ok = all(np.array_equal(A[k], g[k]) for k in ("level", "parent", "child_ptr", "row_start", "perm_row", "perm_col")) and np.array_equal(A["lo"], g["lo"])
    print(name, "tree ok" if ok else "TREE MISMATCH", "nodes", len(A["level"]), "%.3fs" % (time.time() - t0))
    L, Lm = sg.leaf_sets(tree, m["tau"], m["structure"])
    print("  pairs", np.array_equal(np.array(L).reshape(-1, 2), g["L"]), np.array_equal(np.array(Lm).reshape(-1, 2), g["Lm"]))
    if m["structure"] != "h2":
        continue
    spec = sg.KernelSpec(m["kernel"], dx=None if m["kernel"] == "exp" else 0.0)
    M = sg.build_h2(tree, spec, None, None, sg.BuildParams(r=m["r"], tau=m["tau"], basis="interp", rtol=m["rtol"]))
    bad = 0; tot = 0
    for i, f in M.rowfac.items():
        ref = unflatten(g["skel_row_ptr"], g["skel_row"], i)
        tot += 1
        if not np.array_equal(f.skel, ref):
            bad += 1
            if bad <= 3: print("   skel mismatch node", i, f.skel[:8], ref[:8], f.rank, ref.size)
    print("  skeleton mismatches %d / %d, swaps %s" % (bad, tot, M.swaps))
    z = sg.matvec_nodewise(M, g["q"])
    rel = np.linalg.norm(z - g["z"]) / np.linalg.norm(g["z"])
    print("  matvec rel vs reference %.3e" % rel)
