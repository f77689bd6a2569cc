"""The B200 on-line stepper driven by real ROMs from the off-line stage
(reference test cases test_msolver.cpp:87-118, 238-260, 440-465)."""
import numpy as np
import pytest

from paper_1604_06750_b200.fine import FineGrid, SparseVec, make_uniform_medium
from paper_1604_06750_b200.offline import (RomOptions, assemble_nd, assemble_system, build_all_roms,
                                           build_boundary_basis, build_regular, corner_arrays,
                                           regular_partition)
from paper_1604_06750_b200.rom import FlatSystem, RomStepper, system_receiver, system_sources
from paper_1604_06750_b200.signal import Wavelet, steps_for
from tests.helpers import per_trace_rel_l2, rel_l2

pytestmark = pytest.mark.gpu


def _gpu(sys_, corners=False):
    st = RomStepper(FlatSystem.from_system(sys_))
    st.set_sources(system_sources(sys_))
    st.set_receivers(system_receiver(sys_))
    if corners and sys_.corners:
        st.set_corners(*corner_arrays(sys_))
    return st


def test_full_order_1d_rom_equals_fine_on_gpu(gpu_lib, oracle):
    # test_msolver.cpp:87-118: untruncated basis, m = N_i -> exact congruence
    med = make_uniform_medium([19], 1.0, 1.0)
    p = assemble_nd(med)
    part, splits = regular_partition(p, [2])
    opt = RomOptions(m=splits[0].A.shape[0], omega_max=2.5, epsilon_rel=1e-14)
    basis = build_boundary_basis(p, part, opt)
    row = p.node_of((9, 0, 0))
    g = np.zeros(p.n)
    q = np.zeros(p.n)
    g[row] = q[row] = 1.0
    roms = build_all_roms(part, splits, basis, g, q, opt)
    sys_ = assemble_system(part, basis, roms, p.B)
    w = Wavelet(omega_cut=2.5)
    dt = 0.9 * oracle.OracleFine(med).cfl()
    steps = steps_for(500 * dt, dt)
    st = _gpu(sys_)
    st.make_state(dt)
    ws, _ = w.samples_accumulated(dt, steps)
    ms, _ = st.run(steps, ws)
    wf, _ = w.samples_fixed(dt, steps)
    one = [SparseVec(np.array([row], np.int64), np.array([1.0]))]
    fine = FineGrid(med).leapfrog(one, one, dt, steps, wf)[:, 0, 0]
    scale = max(1.0, np.max(np.abs(fine)))
    assert np.max(np.abs(fine - ms[:, 0, 0])) < 1e-10 * scale


def _built_2d():
    opt = RomOptions(m=3, omega_max=4.0, epsilon_rel=1e-3, max_basis_per_interface=4)
    return build_regular([17, 17], 0.5, [2, 2], opt, (8, 4, 0), (8, 12, 0))


def test_real_2d_roms_match_oracle(gpu_lib, oracle):
    b = _built_2d()
    st = _gpu(b.system, corners=True)
    o = oracle.OracleStepper(FlatSystem.from_system(b.system))
    o.set_sources(system_sources(b.system))
    o.set_receivers(system_receiver(b.system))
    o.set_corners(*corner_arrays(b.system))
    dt = 0.5 * o.estimate_dt(1.0)
    w = Wavelet(omega_cut=4.0)
    steps = 200
    ws, _ = w.samples_accumulated(dt, steps)
    for corner in (False, True):
        st.make_state(dt)
        o.make_state(dt)
        tg, _ = st.run(steps, ws, corner=corner)
        to, _ = o.run(steps, ws, corner=corner)
        assert np.max(np.abs(to)) > 0
        assert per_trace_rel_l2(tg, to) < 1e-10
        sg, so = st.get_state(), o.get_state()
        for k in ("u_cur", "ubar_cur"):
            assert rel_l2(sg[k], so[k]) < 1e-10


def test_conjugation_invariant_real_roms(gpu_lib):
    # test_msolver.cpp:238-260
    b = _built_2d()
    st = _gpu(b.system)
    flat = FlatSystem.from_system(b.system)
    st.make_state(0.02)
    w = Wavelet(omega_cut=4.0)
    t = 0.0
    for _ in range(50):
        st.step(w(t))
        t += 0.02
        s = st.get_state()
        for c in range(flat.n_cells):
            for p in range(flat.cell_iface_ptr[c], flat.cell_iface_ptr[c + 1]):
                f = flat.cell_iface_ids[p]
                M = flat.iface_size[f]
                rows = flat.cell_u_off[c] + flat.cell_iface_offsets[p] + np.arange(M)
                assert np.array_equal(s["u_cur"][rows], s["ubar_cur"][flat.iface_row_off[f] + np.arange(M)])


def test_corner_correction_reduces_error(gpu_lib, oracle):
    # test_msolver.cpp:360-385: smooth 2D run, corner correction on vs off
    opt = RomOptions(m=4, omega_max=2.0 * np.pi, epsilon_rel=1e-7)
    b = build_regular([41, 41], 0.05, [2, 2], opt, (20, 10, 0), (20, 30, 0))
    assert b.system.corners
    w = Wavelet(omega_cut=opt.omega_max, delay_factor=5.0)
    med = make_uniform_medium([41, 41], 0.05, 1.0)
    dt = 0.9 * oracle.OracleFine(med).cfl()
    steps = steps_for(6.0, dt)
    src = b.original_pencil.node_of((20, 10, 0))
    rcv = b.original_pencil.node_of((20, 30, 0))
    wf, tf = w.samples_fixed(dt, steps)
    fine = FineGrid(med).leapfrog([SparseVec(np.array([src]), np.array([1.0]))],
                                  [SparseVec(np.array([rcv]), np.array([1.0]))], dt, steps, wf)[:, 0, 0]
    st = _gpu(b.system, corners=True)
    ws, tm = w.samples_accumulated(dt, steps)
    errs = []
    for corner in (False, True):
        st.make_state(dt)
        tr, times = st.run(steps, ws, corner=corner)
        mx, rl = oracle.compare_traces(times, tr[:, 0, 0], tf, fine)
        errs.append(rl)
    assert errs[1] < errs[0]


def test_archive_load_bitwise_and_projected_sources(gpu_lib, oracle, tmp_path):
    # rom_archive.cpp:110-190 + cmd_simulate's load (cli_commands.cpp:111-116)
    from paper_1604_06750_b200.archive import (flat_from_archive, project_receivers, project_sources,
                                               read_rom_archive, write_rom_archive)
    opt = RomOptions(m=3, omega_max=4.0, epsilon_rel=1e-3, max_basis_per_interface=4)
    b = build_regular([17, 17], 0.5, [2, 2], opt, (8, 4, 0), (8, 12, 0))
    d = str(tmp_path / "rom")
    write_rom_archive(d, b.system.roms, b.basis, opt)
    st_a = RomStepper.from_archive(d)
    st_m = _gpu(b.system)
    o = oracle.OracleStepper(FlatSystem.from_system(b.system))
    dt = 0.5 * o.estimate_dt(1.0)
    w, _ = Wavelet(omega_cut=4.0).samples_accumulated(dt, 150)
    for st in (st_a, st_m):
        st.make_state(dt)
    ta, _ = st_a.run(150, w)
    tm, _ = st_m.run(150, w)
    assert np.max(np.abs(tm)) > 0 and np.array_equal(ta, tm)
    # S = 5 new skeleton point sources, R = 3 receivers, projected through the archived S_f
    ar = read_rom_archive(d)
    rng = np.random.default_rng(9)
    pts = rng.choice(np.asarray(b.partition.skeleton), size=8, replace=False)
    G = project_sources(b.partition, ar.basis, [(np.array([k]), np.array([1.0])) for k in pts[:5]])
    rc = project_receivers(b.partition, ar.basis, [(np.array([k]), np.array([1.0])) for k in pts[5:]])
    st_a.set_sources(G)
    st_a.set_receivers(rc)
    ora = oracle.OracleStepper(flat_from_archive(ar))
    ora.set_sources(G)
    ora.set_receivers(rc)
    st_a.make_state(dt)
    ora.make_state(dt)
    tg, _ = st_a.run(150, w)
    to, _ = ora.run(150, w)
    assert np.max(np.abs(to)) > 0
    assert per_trace_rel_l2(tg, to) < 1e-10
