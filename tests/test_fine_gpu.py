"""Bit-exact parity of the sm_100a fine-grid leapfrog with the CPU oracle
(restated fine_leapfrog, reference.cpp:49-80; assemble_nd,
fine_grid.cpp:58-112).  The kernel uses explicitly rounded mul/add/div in
the reference's evaluation order, so traces must be identical."""
import math

import numpy as np
import pytest

from paper_1604_06750_b200._ffi import ConfigError, NumericalError
from paper_1604_06750_b200.fine import (FineGrid, GridMedium, SparseVec, gershgorin_lambda,
                                        make_source, make_uniform_medium, set_receiver)
from paper_1604_06750_b200.signal import Wavelet

pytestmark = pytest.mark.gpu


def _medium(dims, seed, h=0.5):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    return GridMedium(list(dims), h, rng.uniform(1.0, 4.0, n), rng.uniform(1.0, 2.0, n))


@pytest.mark.parametrize("dims,S,R,seed", [
    ((23,), 1, 2, 1),
    ((15, 17), 3, 4, 2),
    ((9, 11, 13), 2, 3, 3),
    ((12, 10, 14), 40, 5, 4),
])
def test_fine_bitexact(gpu_lib, oracle, dims, S, R, seed):
    med = _medium(dims, seed)
    rng = np.random.default_rng(seed)
    nd = len(dims)

    def rnd_loc():
        return tuple(int(rng.integers(1, d - 1)) for d in dims) + (0,) * (3 - nd)

    kinds = ["point", "unit_impulse", "taper"]
    sources = [make_source(list(dims), rnd_loc(), kind=kinds[s % 3], rho=med.rho, taper_axis=0,
                           taper_halfwidth=1.5) for s in range(S)]
    receivers = [set_receiver(list(dims), rnd_loc()) for _ in range(R)]
    ora = oracle.OracleFine(med)
    dt = 0.5 * ora.cfl()
    steps = 90
    w, _ = Wavelet(kind="ricker", omega_cut=0.5 / dt).samples_fixed(dt, steps)
    tg = FineGrid(med).leapfrog(sources, receivers, dt, steps, w)
    to = ora.leapfrog(sources, receivers, dt, steps, w)
    assert np.max(np.abs(to)) > 0.0
    assert np.array_equal(tg, to)


def test_fine_per_source_wavelets(gpu_lib, oracle):
    dims = (10, 11, 12)
    med = _medium(dims, 7)
    rng = np.random.default_rng(7)
    S = 6
    sources = [make_source(list(dims), (1 + s, 2, 3)) for s in range(S)]
    receivers = [set_receiver(list(dims), (4, 5, 6)), set_receiver(list(dims), (2, 2, 2))]
    ora = oracle.OracleFine(med)
    dt = 0.4 * ora.cfl()
    w = rng.standard_normal((50, S))
    assert np.array_equal(FineGrid(med).leapfrog(sources, receivers, dt, 50, w),
                          ora.leapfrog(sources, receivers, dt, 50, w))


def test_fine_instability(gpu_lib, oracle):
    med = make_uniform_medium([9, 9], 1.0, 1.0)
    src = [make_source([9, 9], (4, 4, 0))]
    rcv = [set_receiver([9, 9], (4, 4, 0))]
    w, _ = Wavelet(omega_cut=3.0).samples_fixed(2.0, 100)
    msgs = []
    for runner in (FineGrid(med), oracle.OracleFine(med)):
        with pytest.raises(NumericalError, match="fine_leapfrog: instability at step") as ei:
            runner.leapfrog(src, rcv, 2.0, 100, w)
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]


def test_fine_zero_source(gpu_lib):
    med = make_uniform_medium([9, 9], 0.5, 1.0)
    tr = FineGrid(med).leapfrog([SparseVec(np.zeros(0, np.int64), np.zeros(0))],
                                [SparseVec(np.array([10], np.int64), np.array([1.0]))], 0.05, 40,
                                np.ones(40))
    assert np.all(tr == 0.0)


def test_fine_rejects_bad_input(gpu_lib):
    med = make_uniform_medium([9, 9], 0.5, 1.0)
    g = FineGrid(med)
    with pytest.raises(ConfigError):
        g.leapfrog([SparseVec(np.array([10**6], np.int64), np.array([1.0]))], [], 0.05, 4, np.ones(4))
    with pytest.raises(ConfigError):
        g.leapfrog([make_source([9, 9], (4, 4, 0))], [], -0.05, 4, np.ones(4))
