"""e2e pipeline probe: MatvecStream per-step time vs depth / flush (cfg2, 16 RHS)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.workloads import CONFIGS, build_params, make_points
c = CONFIGS[2]
X, Y, rng = make_points(2)
spec, params = build_params(2)
R = 16
q = rng.standard_normal((X.shape[0], R))
tree = sg.build_tree(sg.PointSet(torch.from_numpy(X).cuda()), nu0=c["nu0"], mode=c["mode"], tau=c["tau"])
M = sg.build_h2(tree, spec, None, None, params)
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
q_pin = [torch.from_numpy(q.copy()).pin_memory() for _ in range(3)]
z_pin = [torch.empty((M.n_row, R), dtype=torch.float64).pin_memory() for _ in range(3)]
for depth in (2, 3):
    for K in (10, 40):
        for fl in (True, False):
            pipe = sg.MatvecStream(M, R, depth=depth)
            for i in range(3):
                pipe.submit(q_pin[i % depth], z_pin[i % depth])
            pipe.synchronize(); torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(pipe.s_in)
            for i in range(K):
                pipe.submit(q_pin[i % depth], z_pin[i % depth], before=flush.zero_ if fl else None)
            s1.record(pipe.s_out); s1.synchronize()
            print("depth %d K %d flush %d: %.3f ms/step" % (depth, K, fl, s0.elapsed_time(s1) / K))
Q = torch.from_numpy(q).cuda(); Z = torch.empty_like(Q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(5):
    e0.record(); sg.matvec_device(M, Q, Z); e1.record(); e1.synchronize()
print("device matvec %.3f ms" % e0.elapsed_time(e1))
t0 = time.perf_counter()
for i in range(20):
    pipe.submit(q_pin[i % 3], z_pin[i % 3])
t1 = time.perf_counter(); pipe.synchronize()
print("host submit cost %.3f ms/step" % ((t1 - t0) / 20 * 1e3))
