"""Host-side logic of the drop-in package that needs no GPU."""

import numpy as np
import pytest

import paper_1705_05443_b200 as sg
from oracle import smash_oracle as orc
from paper_1705_05443_b200.workloads import CONFIGS, make_points


def test_well_separated_known_answers():
    a = sg.Box.of((0.0,), (1.0,))
    b = sg.Box.of((2.0,), (3.0,))
    assert sg.well_separated(a, b, 0.5)
    assert not sg.well_separated(a, a, 0.5)
    c = sg.Box.of((1.0,), (2.0,))
    assert not sg.well_separated(a, c, 0.5) and sg.well_separated(a, c, 1.0)


def test_well_separated_matches_oracle_fma_geometry():
    rng = np.random.default_rng(0)
    lo = rng.random((400, 2))
    hi = lo + rng.random((400, 2)) * 0.3
    lo2 = rng.random((400, 2))
    hi2 = lo2 + rng.random((400, 2)) * 0.3
    ref = orc.separated(lo, hi, lo2, hi2, 0.7)
    got = [sg.well_separated(sg.Box.of(lo[i], hi[i]), sg.Box.of(lo2[i], hi2[i]), 0.7) for i in range(400)]
    assert np.array_equal(np.array(got), ref)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_workload_generators_match_oracle(cfg):
    n = 1000
    X, Y, rng = make_points(cfg, N=n)
    Xo, Yo, rngo = orc.make_config_points(cfg, N=n)
    assert np.array_equal(X, Xo) and np.array_equal(Y, Yo)
    assert np.array_equal(rng.standard_normal(5), rngo.standard_normal(5))
    assert CONFIGS[cfg]["r"] == orc.CONFIGS[cfg]["r"]


def test_kernel_spec_validation():
    with pytest.raises(ValueError):
        sg.KernelSpec("laplace_dlp")
    with pytest.raises(ValueError):
        sg.KernelSpec("nope")
    assert sg.KernelSpec("exp").dx_value == 1.0
    assert sg.KernelSpec("log").dx_value == 0.0


def test_point_set_shapes():
    P = sg.PointSet(np.arange(6.0).reshape(3, 2))
    assert P.n == 3 and P.dim == 2
    assert sg.PointSet([1.0, 2.0]).n == 1
