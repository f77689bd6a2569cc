"""Parity at BASELINE.json's full sizes (config 3: 16^3 cells, M = 6,
S = 64; config 5: 16^3 cells of 24^3, M = 17; the 257^3 fine grid).

The oracle cannot run these configurations to completion inside a test, so
the full-size runs are pinned by properties that do not depend on size:
  * oracle parity on a source subset over a short window of the FULL system
    (rel. L2 <= 1e-10, the north-star gate; the fine grid bit-exact);
  * exact linearity: doubling the wavelet doubles every trace sample
    bitwise (every operation on the path is linear, and x2 is exact in
    binary floating point);
  * source independence: the first sources of an S = 64 run equal, bitwise,
    a run with only those sources (different source tiling, same bits);
  * zero in -> zero out over the full system, exactly.
"""
import math

import numpy as np
import pytest

from paper_1604_06750_b200.rom import RomStepper
from paper_1604_06750_b200.signal import Wavelet
from paper_1604_06750_b200.synthetic import CONFIGS, config_case
from tests.helpers import per_trace_rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _rom(case, g):
    st = RomStepper(case.flat)
    st.set_sources(np.ascontiguousarray(g))
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    return st


@pytest.fixture(scope="module")
def c3():
    return config_case("c3", S=64)


@pytest.fixture(scope="module")
def c3_run(c3):
    steps = 200
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(c3.dt, steps)
    st = _rom(c3, c3.g)
    tr, _ = st.run(steps, w)
    st.close()
    return steps, w, tr


def test_c3_full_system_oracle_subset(gpu_lib, oracle, c3, c3_run):
    """Two of the 64 sources through the oracle restatement, 40 steps of the
    full 4096-cell system; the GPU ran all 64 together."""
    _, w, tr = c3_run
    steps = 40
    ora = oracle.OracleStepper(c3.flat)
    ora.set_sources(np.ascontiguousarray(c3.g[:, :2]))
    ora.set_receivers(c3.receivers)
    ora.make_state(c3.dt)
    to, _ = ora.run(steps, w[:steps], threads=2)
    assert np.abs(to).max() > 0
    assert per_trace_rel_l2(tr[:steps + 1, :, :2], to) < TOL


def test_c3_exact_linearity(gpu_lib, c3, c3_run):
    steps, w, tr = c3_run
    st = _rom(c3, c3.g)
    tr2, _ = st.run(steps, 2.0 * w)
    st.close()
    assert np.abs(tr).max() > 0
    assert np.array_equal(tr2, 2.0 * tr)


def test_c3_source_subset_bitwise(gpu_lib, c3, c3_run):
    steps, w, tr = c3_run
    st = _rom(c3, c3.g[:, :8])
    tr8, _ = st.run(steps, w)
    st.close()
    assert np.array_equal(tr8, tr[:, :, :8])


def test_c3_zero_in_zero_out(gpu_lib, c3):
    st = _rom(c3, np.zeros_like(c3.g))
    tr, _ = st.run(50, np.ones(50))
    s = st.get_state()
    st.close()
    assert not np.any(tr) and not np.any(s["u_cur"]) and not np.any(s["ubar_cur"])


def test_c5_full_system_oracle_subset_and_linearity(gpu_lib, oracle):
    """Config 5 (ktilde = 102, the K-streaming kernel family) at S = 8."""
    case = config_case("c5", S=8)
    steps = 60
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, steps)
    st = _rom(case, case.g)
    tr, _ = st.run(steps, w)
    st.make_state(case.dt)
    tr2, _ = st.run(steps, 2.0 * w)
    st.close()
    assert np.array_equal(tr2, 2.0 * tr)
    sub = 20
    ora = oracle.OracleStepper(case.flat)
    ora.set_sources(np.ascontiguousarray(case.g[:, :1]))
    ora.set_receivers(case.receivers)
    ora.make_state(case.dt)
    to, _ = ora.run(sub, w[:sub])
    assert np.abs(to).max() > 0
    assert per_trace_rel_l2(tr[:sub + 1, :, :1], to) < TOL


def test_fine_c3_grid_bitexact_subset(gpu_lib, oracle):
    """257^3 fine grid (16.6 M interior nodes), seeded lognormal medium:
    S = 64 sources on the GPU; the first two are bit-identical to an S = 2
    GPU run and that to the oracle over 3 steps."""
    from paper_1604_06750_b200.fine import FineGrid, SparseVec, gershgorin_lambda, node_of
    from paper_1604_06750_b200.synthetic import lognormal_medium, skeleton_points

    c = CONFIGS["c3"]
    dims = list(c["fine_dims"])
    med = lognormal_medium(dims, seed=77)
    dt = 0.5 * 2.0 / math.sqrt(gershgorin_lambda(med))
    S = 64
    pts = skeleton_points(dims, c["cell_len"], S, seed=5)
    vec = lambda p: SparseVec(np.array([node_of(dims, p)], np.int64), np.array([1.0]))
    src = [vec(p) for p in pts]
    # receivers on every source node and next to the first two (a 3-step
    # stencil front reaches 3 nodes)
    near = [tuple(int(x) + (1 if a == 0 else 0) for a, x in enumerate(p)) for p in pts[:2]]
    rcv = [vec(p) for p in pts] + [vec(p) for p in near]
    steps = 3
    # a wavelet that is nonzero from the first step, so 3 steps move data
    w = np.array([1.0, -0.5, 0.25])
    fg = FineGrid(med)
    t64 = fg.leapfrog(src, rcv, dt, steps, w)
    t2 = fg.leapfrog(src[:2], rcv, dt, steps, w)
    fg.close()
    assert np.abs(t2).max() > 0
    assert np.array_equal(t64[:, :, :2], t2)
    of = oracle.OracleFine(med)
    to = of.leapfrog(src[:2], rcv, dt, steps, w, threads=2)
    assert np.array_equal(t2, to)
