"""BASELINE.json configurations as seeded synthetic workloads.

No public dataset is named by BASELINE; every input is drawn with
``np.random.default_rng(seed = config id)`` in the documented order, and the
right-hand sides are drawn after the points from the same generator.
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(name="hss_log_1d", structure="hss", kernel="log", dim=1, mode="binary", nu0=64, r=10,
            tau=0.6, rtol=1e-8, eps_svd=1e-9, nrhs=(1,), N=4096),
    2: dict(name="h2_invr_2d", structure="h2", kernel="inv_r", dim=2, mode="2d", nu0=64, r=36,
            tau=0.7, rtol=1e-8, eps_svd=0.0, nrhs=(1, 16), N=2 ** 17),
    3: dict(name="h2_exp_3d", structure="h2", kernel="exp", dim=3, mode="2d", nu0=128, r=125,
            tau=0.7, rtol=1e-6, eps_svd=0.0, nrhs=(1,), N=2 ** 20),
    4: dict(name="hss_cauchy_1d", structure="hss", kernel="cauchy", dim=1, mode="binary", nu0=128,
            r=16, tau=0.6, rtol=1e-10, eps_svd=1e-11, nrhs=(8,), N=2 ** 20),
    5: dict(name="h2_log_2d_nonuniform", structure="h2", kernel="log", dim=2, mode="2d", nu0=64,
            r=64, tau=0.7, rtol=1e-8, eps_svd=0.0, nrhs=(16,), N=2 ** 21),
}


def make_points(cfg: int, N: int = None, seed: int = None):
    """(X, Y, rng): Y is X for the symmetric configs; rng continues after the points."""
    c = CONFIGS[cfg]
    N = c["N"] if N is None else N
    rng = np.random.default_rng(cfg if seed is None else seed)
    if cfg in (1, 2, 3):
        X = rng.random((N, c["dim"]))
        return X, X, rng
    if cfg == 4:
        X = (np.arange(N, dtype=np.float64) / N).reshape(-1, 1)
        Y = ((np.arange(N, dtype=np.float64) + 0.5) / N).reshape(-1, 1)
        return X, Y, rng
    if cfg == 5:
        h = N // 2
        ang = rng.random(h) * 2 * np.pi
        rad = 1 + rng.normal(0, 1e-3, h)
        circle = np.column_stack([rad * np.cos(ang), rad * np.sin(ang)])
        centres = rng.random((4, 2))
        lab = rng.integers(0, 4, N - h)
        off = rng.normal(0, 0.02, (N - h, 2))
        X = np.vstack([circle, centres[lab] + off])
        return X, X, rng
    raise ValueError("unknown config %r" % cfg)


def build_params(cfg: int):
    """(KernelSpec, BuildParams) of a config for this package."""
    from .hss import BuildParams
    from .kernel import KernelSpec
    c = CONFIGS[cfg]
    spec = KernelSpec(c["kernel"], dx=None if c["kernel"] == "exp" else 0.0)
    return spec, BuildParams(r=c["r"], tau=c["tau"], eps_svd=c["eps_svd"], s=2.0, basis="interp",
                             rtol=c["rtol"])
