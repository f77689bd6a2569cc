"""Off-line restatement checked against the reference's own KATs
(proj/tests/test_romgen.cpp, test_partition.cpp, test_msolver.cpp) and the
on-line oracle driven by real (not synthetic) ROMs.  CPU only."""
import math

import numpy as np
import pytest

from paper_1604_06750_b200.fine import GridMedium, make_uniform_medium
from paper_1604_06750_b200.offline import (RomOptions, assemble_nd, assemble_system, build_all_roms,
                                           build_boundary_basis, build_regular, corner_arrays,
                                           evaluate_sfraction, regular_partition, remove_corner_set,
                                           resolvent_transfer, sfraction_coeffs)
from paper_1604_06750_b200.offline.romgen import block_lanczos, project_pencil, rational_krylov
from paper_1604_06750_b200.rom import FlatSystem, system_receiver, system_sources
from paper_1604_06750_b200.signal import Wavelet, steps_for


def _oracle_for(oracle, sys):
    o = oracle.OracleStepper(FlatSystem.from_system(sys))
    o.set_sources(system_sources(sys))
    o.set_receivers(system_receiver(sys))
    return o


def test_uniform_1d_cell_ladders():
    # test_romgen.cpp:323-341: Lhat = [2, 1, ..., 1], L = [1, ..., 1]
    p = assemble_nd(make_uniform_medium([19], 1.0, 1.0))
    part, splits = regular_partition(p, [2])
    cell = splits[0]
    n = cell.A.shape[0]
    bl = np.searchsorted(part.cells[0], part.boundaries[0])
    PS = np.zeros((n, 1))
    PS[bl[0], 0] = 1.0
    V = rational_krylov(cell, PS, -0.8, n)
    Am, Bm, Sm = project_pencil(cell, V, PS)
    T, beta1 = block_lanczos(Am, Bm, Sm, n, 1)
    hat, main = sfraction_coeffs(T, beta1, n, 1)
    assert hat[0][0, 0] == pytest.approx(2.0, rel=1e-8)
    for k in range(1, n):
        assert hat[k][0, 0] == pytest.approx(1.0, rel=1e-7)
    for k in range(n):
        assert main[k][0, 0] == pytest.approx(1.0, rel=1e-7)


def test_triple_equality_on_built_roms():
    # test_romgen.cpp:396-431 (S-fraction vs block resolvent, SPD ladders)
    med = make_uniform_medium([17, 9], 0.5, 1.0)
    med.sigma = 1.0 + 0.4 * np.sin(0.31 * np.arange(med.sigma.size))
    p = assemble_nd(med)
    part, splits = regular_partition(p, [2, 1])
    opt = RomOptions(m=3, omega_max=4.0, epsilon_rel=1e-8)
    basis = build_boundary_basis(p, part, opt)
    g = np.zeros(p.n)
    q = np.zeros(p.n)
    g[part.skeleton[0]] = 1.0
    q[part.skeleton[1]] = 1.0
    roms = build_all_roms(part, splits, basis, g, q, opt)
    rng = np.random.default_rng(2024)
    for rom in roms:
        for L in list(rom.ladder_hat) + list(rom.ladder):
            assert np.linalg.eigvalsh(L).min() > 0.0
        for _ in range(10):
            w2 = complex(rng.uniform(-5, 5), rng.uniform(0.1, 3))
            a = evaluate_sfraction(rom.ladder_hat, rom.ladder, w2)
            b = resolvent_transfer(rom.T, rom.beta1, w2)
            scale = max(1e-30, np.max(np.abs(a)))
            assert np.max(np.abs(a - b)) < 1e-9 * scale


def test_regular_partition_weights_2x2():
    # test_partition.cpp:282-313
    p = assemble_nd(make_uniform_medium([9, 9], 1.0, 1.0))
    part, splits = regular_partition(p, [2, 2])
    assert part.num_cells() == 4
    center = p.node_of((4, 4))
    assert center in set(part.corner_set.tolist())
    f01 = part.interfaces[0]
    assert f01.ci == 0
    cell0 = part.cells[0]
    pos = np.searchsorted(cell0, p.node_of((4, 2)))
    post = np.searchsorted(cell0, p.node_of((4, 1)))
    assert splits[0].A[pos, post] == pytest.approx(0.5)
    assert splits[0].B[pos] == pytest.approx(0.5)
    posi = np.searchsorted(cell0, p.node_of((2, 2)))
    assert splits[0].A[posi, posi] == pytest.approx(-4.0)
    assert splits[0].B[posi] == pytest.approx(1.0)


def test_corner_removal_2x2_hanging_copies():
    # test_partition.cpp:315-362
    p = assemble_nd(make_uniform_medium([9, 9], 1.0, 1.0))
    part, splits = regular_partition(p, [2, 2])
    center = p.node_of((4, 4))
    pm, pt, sp_ = remove_corner_set(p, part, splits)
    assert pt.corner_set.size == 0
    assert len(pt.hanging) == 4
    assert pm.n == p.n + 3
    assert all(h.parent == center for h in pt.hanging)
    masses = [pm.B[h.id] for h in pt.hanging]
    assert masses == pytest.approx([0.5] * 4)
    assert pm.B.sum() == pytest.approx(p.B.sum() + p.B[center])
    D = (pm.A - pm.A.T).tocoo()
    assert np.max(np.abs(D.data)) == 0.0 if D.nnz else True
    for a in range(len(pt.interfaces)):
        for b in range(a + 1, len(pt.interfaces)):
            assert np.intersect1d(pt.interfaces[a].nodes, pt.interfaces[b].nodes).size == 0


def test_two_1d_cells_shared_mass():
    # test_msolver.cpp:40-49: mass = 1 / (1/l1 + 1/l2)
    b = build_regular([17], 1.0, [2], RomOptions(m=3, omega_max=3.0), (8, 0, 0), (8, 0, 0))
    assert len(b.system.ifaces) == 1
    l1 = b.system.roms[0].ladder_hat[0][0, 0]
    l2 = b.system.roms[1].ladder_hat[0][0, 0]
    assert b.system.ifaces[0].mass[0, 0] == pytest.approx(1.0 / (1.0 / l1 + 1.0 / l2))


def test_full_order_1d_rom_equals_fine_leapfrog_oracle(oracle):
    # test_msolver.cpp:87-118 on the CPU oracle (ROM stepper vs fine leapfrog)
    p = assemble_nd(make_uniform_medium([19], 1.0, 1.0))
    part, splits = regular_partition(p, [2])
    opt = RomOptions(m=splits[0].A.shape[0], omega_max=2.5, epsilon_rel=1e-14)
    basis = build_boundary_basis(p, part, opt)
    g = np.zeros(p.n)
    q = np.zeros(p.n)
    g[p.node_of((9, 0, 0))] = 1.0
    q[p.node_of((9, 0, 0))] = 1.0
    roms = build_all_roms(part, splits, basis, g, q, opt)
    sys_ = assemble_system(part, basis, roms, p.B)
    w = Wavelet(omega_cut=2.5)
    med = make_uniform_medium([19], 1.0, 1.0)
    of = oracle.OracleFine(med)
    dt = 0.9 * of.cfl()
    steps = steps_for(500 * dt, dt)
    o = _oracle_for(oracle, sys_)
    o.make_state(dt)
    ws, _ = w.samples_accumulated(dt, steps)
    ms, _ = o.run(steps, ws)
    from paper_1604_06750_b200.fine import SparseVec
    wf, _ = w.samples_fixed(dt, steps)
    row = p.node_of((9, 0, 0))
    fine = of.leapfrog([SparseVec(np.array([row]), np.array([1.0]))],
                       [SparseVec(np.array([row]), np.array([1.0]))], dt, steps, wf)[:, 0, 0]
    scale = max(1.0, np.max(np.abs(fine)))
    assert np.max(np.abs(fine - ms[:, 0, 0])) < 1e-10 * scale


def test_real_2d_rom_oracle_invariants(oracle):
    # test_msolver.cpp:238-301 with real ROMs (energy, conjugation, reversal)
    opt = RomOptions(m=3, omega_max=4.0, epsilon_rel=1e-3, max_basis_per_interface=4)
    b = build_regular([17, 17], 0.5, [2, 2], opt, (8, 4, 0), (8, 12, 0))
    o = _oracle_for(oracle, b.system)
    o.set_sources(np.zeros_like(system_sources(b.system)))
    dt = 0.5 * o.estimate_dt(1.0)
    o.make_state(dt)
    rng = np.random.default_rng(77)
    st = o.get_state()
    init = {k: rng.uniform(-0.2, 0.2, size=st[k].shape) for k in ("u_cur", "u_prev", "ubar_cur", "ubar_prev")}
    o.set_state(**init)
    e0 = o.energy()
    drift = 0.0
    for _ in range(300):
        o.step(0.0)
        drift = max(drift, float(np.max(np.abs(o.energy() - e0) / np.abs(e0))))
    assert drift < 1e-8


def test_corner_correction_reduces_error_oracle(oracle):
    # test_msolver.cpp:360-385 on the oracle
    from paper_1604_06750_b200.fine import SparseVec
    opt = RomOptions(m=4, omega_max=2.0 * np.pi, epsilon_rel=1e-7)
    b = build_regular([41, 41], 0.05, [2, 2], opt, (20, 10, 0), (20, 30, 0))
    assert b.system.corners
    w = Wavelet(omega_cut=opt.omega_max, delay_factor=5.0)
    med = make_uniform_medium([41, 41], 0.05, 1.0)
    of = oracle.OracleFine(med)
    dt = 0.9 * of.cfl()
    steps = steps_for(6.0, dt)
    src = b.original_pencil.node_of((20, 10, 0))
    rcv = b.original_pencil.node_of((20, 30, 0))
    wf, tf = w.samples_fixed(dt, steps)
    fine = of.leapfrog([SparseVec(np.array([src]), np.array([1.0]))],
                       [SparseVec(np.array([rcv]), np.array([1.0]))], dt, steps, wf)[:, 0, 0]
    o = _oracle_for(oracle, b.system)
    o.set_corners(*corner_arrays(b.system))
    ws, _ = w.samples_accumulated(dt, steps)
    errs = []
    for corner in (False, True):
        o.make_state(dt)
        tr, times = o.run(steps, ws, corner=corner)
        errs.append(oracle.compare_traces(times, tr[:, 0, 0], tf, fine)[1])
    assert errs[1] < errs[0]
