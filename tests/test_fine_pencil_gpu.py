"""fine_cfl (reference.cpp:24-47) and fine_leapfrog on an assembled
SparsePencil (msw_fine_create_csc / msw_fine_cfl) on the B200.

Tolerances: fine_cfl is a power iteration whose stopping rule is itself a
1e-7 relative change of the eigenvalue estimate, and its dot products are
summed in a different (deterministic) order than Eigen's, so dt is compared
with the oracle at 1e-6 relative; the reference's own KATs at their stated 1%
(test_reference.cpp:68-85) and 5% (test_msolver.cpp:213-236).  Leapfrog
traces on a pencil are bit-identical (rows summed in Eigen's column order).
"""
import math

import numpy as np
import pytest

from paper_1604_06750_b200.fine import FineGrid, GridMedium, SparseVec, make_uniform_medium
from paper_1604_06750_b200.offline import (RomOptions, assemble_nd, assemble_system, build_all_roms,
                                           build_boundary_basis, build_regular, regular_partition)
from paper_1604_06750_b200.rom import FlatSystem, RomStepper, system_receiver, system_sources

pytestmark = pytest.mark.gpu


def _cfl_pencil(med):
    fg = FineGrid.from_pencil(assemble_nd(med))
    dt = fg.cfl()
    fg.close()
    return dt


def _cfl_medium(med):
    fg = FineGrid(med)
    dt = fg.cfl()
    fg.close()
    return dt


def test_fine_cfl_known_spectra(gpu_lib):
    # test_reference.cpp:68-85
    m1 = make_uniform_medium([41], 0.25, 1.0)
    d1 = _cfl_pencil(m1)
    assert d1 == pytest.approx(0.25, rel=0.01)
    m4 = make_uniform_medium([41], 0.25, 4.0)
    assert _cfl_pencil(m4) / d1 == pytest.approx(0.5, rel=0.01)
    # 2-D: the reference compares with a dense eigensolve of -A
    m2 = make_uniform_medium([21, 21], 0.5, 1.3)
    p2 = assemble_nd(m2)
    lam = np.linalg.eigvalsh(-p2.A.toarray()).max()
    assert _cfl_pencil(m2) == pytest.approx(2.0 / math.sqrt(lam), rel=0.01)
    assert _cfl_medium(m2) == pytest.approx(_cfl_pencil(m2), rel=1e-9)


@pytest.mark.parametrize("dims,h,seed", [([40], 0.5, 1), ([23, 19], 1.0, 2), ([14, 12, 17], 0.7, 3)])
def test_fine_cfl_matches_oracle(gpu_lib, oracle, dims, h, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    med = GridMedium(list(dims), h, rng.uniform(0.5, 3.0, n), rng.uniform(1.0, 2.0, n))
    ref = oracle.OracleFine(med).cfl()
    assert _cfl_medium(med) == pytest.approx(ref, rel=1e-6)
    assert _cfl_pencil(med) == pytest.approx(ref, rel=1e-6)


def test_estimate_dt_within_5pct_of_fine_cfl(gpu_lib):
    # test_msolver.cpp:213-236 through the product (msw_estimate_dt,
    # msw_fine_cfl): two-cell 1-D full-order ROM, m = N_i
    def dts(sigma):
        med = make_uniform_medium([19], 1.0, sigma)
        p = assemble_nd(med)
        part, splits = regular_partition(p, [2])
        opt = RomOptions(m=splits[0].A.shape[0], omega_max=2.5)
        basis = build_boundary_basis(p, part, opt)
        row = p.node_of((9, 0, 0))
        g = np.zeros(p.n)
        q = np.zeros(p.n)
        g[row] = q[row] = 1.0
        sys_ = assemble_system(part, basis, build_all_roms(part, splits, basis, g, q, opt), p.B)
        st = RomStepper(FlatSystem.from_system(sys_))
        st.set_sources(system_sources(sys_))
        st.set_receivers(system_receiver(sys_))
        est = st.estimate_dt(1.0)
        st.close()
        fg = FineGrid.from_pencil(p)
        fc = fg.cfl()
        fg.close()
        return est, fc

    est1, fc1 = dts(1.0)
    assert est1 == pytest.approx(fc1, rel=0.05)
    est4, _ = dts(4.0)
    assert est4 < est1


def test_pencil_path_bitexact_vs_medium_and_oracle(gpu_lib, oracle):
    rng = np.random.default_rng(11)
    dims = [13, 11, 12]
    n = int(np.prod(dims))
    med = GridMedium(dims, 0.5, rng.uniform(1.0, 3.0, n), rng.uniform(1.0, 2.0, n))
    p = assemble_nd(med)
    dt = 0.5 * _cfl_medium(med)
    src = [SparseVec(np.array([p.node_of((6, 5, 6))], np.int64), np.array([1.0])),
           SparseVec(np.array([p.node_of((3, 4, 8)), p.node_of((3, 4, 9))], np.int64), np.array([0.5, -0.25]))]
    rcv = [SparseVec(np.array([p.node_of((7, 5, 6))], np.int64), np.array([1.0])),
           SparseVec(np.array([p.node_of((4, 4, 8))], np.int64), np.array([2.0]))]
    steps = 60
    w = np.sin(0.3 * np.arange(steps)) * np.exp(-0.01 * np.arange(steps))
    fp = FineGrid.from_pencil(p)
    tp = fp.leapfrog(src, rcv, dt, steps, w)
    fp.close()
    fm = FineGrid(med)
    tm = fm.leapfrog(src, rcv, dt, steps, w)
    fm.close()
    to = oracle.OracleFine(med).leapfrog(src, rcv, dt, steps, w)
    assert np.abs(tp).max() > 0
    assert np.array_equal(tp, tm)
    assert np.array_equal(tp, to)


def test_corner_modified_pencil_bitexact_vs_oracle(gpu_lib, oracle):
    """The pencil after remove_corner_set (hanging copies appended, rows not
    on a regular grid) -- only the general path can run it."""
    opt = RomOptions(m=3, omega_max=4.0, epsilon_rel=1e-3, max_basis_per_interface=4)
    b = build_regular([17, 17], 0.5, [2, 2], opt, (8, 4, 0), (8, 12, 0))
    p = b.pencil
    assert p.n > b.original_pencil.n  # hanging copies present
    A = p.A.tocsr()
    A.sort_indices()
    ora = oracle.OracleFine(csr=(p.n, A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data, p.B))
    dt = 0.5 * ora.cfl()
    fg = FineGrid.from_pencil(p)
    assert fg.cfl() == pytest.approx(ora.cfl(), rel=1e-6)
    gi = int(np.nonzero(b.g)[0][0])
    qi = int(np.nonzero(b.q)[0][0])
    hang = p.n - 1  # a hanging copy row
    src = [SparseVec(np.array([gi], np.int64), np.array([1.0]))]
    rcv = [SparseVec(np.array([qi], np.int64), np.array([1.0])),
           SparseVec(np.array([hang], np.int64), np.array([1.0]))]
    steps = 200
    w = np.sin(0.2 * np.arange(steps))
    tg = fg.leapfrog(src, rcv, dt, steps, w)
    fg.close()
    to = ora.leapfrog(src, rcv, dt, steps, w)
    assert np.abs(tg).max() > 0
    assert np.array_equal(tg, to)
