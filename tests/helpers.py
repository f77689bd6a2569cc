"""Shared fixtures for parity tests: reference-shaped hand-built systems
(proj/tests/test_helpers.hpp) and comparison metrics (trace_io.cpp:36-67)."""
import numpy as np

from paper_1604_06750_b200.rom import (CornerCopy, CornerGroup, CoupledInterface, FlatSystem,
                                       MultiscaleSystem, SubdomainROM)


def scalar_oscillator(lhat, lmain):
    """test_helpers.hpp:48-76: one cell, one single-sided interface, m = 1,
    ktilde = 1, u'' = -(L * mass) u, mass = lhat."""
    rom = SubdomainROM(cell=0, m=1, ktilde=1, shift=-1.0, iface_ids=[0], iface_offsets=[0, 1],
                       ladder_hat=[np.full((1, 1), lhat)], ladder=[np.full((1, 1), lmain)],
                       g_proj=[np.ones(1)], q_proj=[np.ones(1)])
    cf = CoupledInterface(part_iface=0, ci=0, cj=-1, li=0, lj=-1, size=1, S=np.eye(1),
                          mass_form=np.full((1, 1), 1.0 / lhat), mass=np.full((1, 1), lhat),
                          g_proj=np.ones(1), q_proj=np.ones(1))
    return MultiscaleSystem(roms=[rom], ifaces=[cf])


def corner_fixture():
    """test_msolver.cpp:303-358: two single-sided 2-row interfaces on one
    placeholder m=1 cell, one corner group with copies (iface 0,row 0) and
    (iface 1,row 1)."""
    ifaces = []
    for f in range(2):
        ifaces.append(CoupledInterface(part_iface=f, ci=0, cj=-1, li=f, lj=-1, size=2, S=np.eye(2),
                                       mass=np.eye(2), mass_form=np.eye(2), g_proj=np.zeros(2),
                                       q_proj=np.zeros(2)))
    rom = SubdomainROM(cell=0, m=1, ktilde=4, iface_ids=[0, 1], iface_offsets=[0, 2, 4],
                       ladder=[np.eye(4)], ladder_hat=[np.eye(4)])
    sys = MultiscaleSystem(roms=[rom], ifaces=ifaces,
                           corners=[CornerGroup(0, [CornerCopy(0, 0, 1.0), CornerCopy(1, 1, 1.0)])])
    return sys


def corner_arrays(sys):
    grp_ptr, ci, cr, cm = [0], [], [], []
    for g in sys.corners:
        for c in g.copies:
            ci.append(c.iface)
            cr.append(c.row)
            cm.append(c.mass)
        grp_ptr.append(len(ci))
    iface_K = [f.S.shape[0] for f in sys.ifaces]
    basis = np.concatenate([np.asarray(f.S, np.float64).T.reshape(-1) for f in sys.ifaces])
    return grp_ptr, ci, cr, cm, iface_K, basis


def rel_l2(a, b):
    """compare_traces' rel_l2 on identical grids (trace_io.cpp:193-203)."""
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    num = np.sum((a - b) ** 2)
    den = np.sum(b ** 2)
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))


def per_trace_rel_l2(a, b):
    """max over (receiver, source) traces of rel_l2, a/b [steps+1, R, S]."""
    worst = 0.0
    for r in range(a.shape[1]):
        for s in range(a.shape[2]):
            worst = max(worst, rel_l2(a[:, r, s], b[:, r, s]))
    return worst
