"""Evaluate one 1024x1024 kernel block per kernel kind (for ncu DP-op counts -> c_K)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1705_05443_b200 as sg
from paper_1705_05443_b200.kernel import kernel_block_coords
rng = np.random.default_rng(0)
for kind, d in (("inv_r", 2), ("log", 2), ("exp", 3), ("cauchy", 1)):
    X = rng.random((1024, d)); Y = rng.random((1024, d)) + 2.0
    K = kernel_block_coords(sg.KernelSpec(kind, dx=0.0), X, Y)
    print(kind, K.shape, float(K[0, 0]))
