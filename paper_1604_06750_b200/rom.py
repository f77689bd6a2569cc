"""Host-side ROM system types and the device stepper handle.

Python mirror of the reference's on-line types (proj/include/mswave):
  SubdomainROM      romgen.hpp:23-45
  CoupledInterface  msolver.hpp:16-25
  CornerGroup       msolver.hpp:28-36
  MultiscaleSystem  msolver.hpp:38-46
plus ``FlatSystem`` (the plain-array form handed to the C ABI, see
include/mswave_b200.h ``msw_system_desc``) and ``RomStepper`` (the
device-resident system: ``msw_create`` ... ``msw_run``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _ffi
from ._ffi import ConfigError, NumericalError, ptr


# ---------------------------------------------------------------------------
# reference-shaped types
# ---------------------------------------------------------------------------

@dataclass
class SubdomainROM:
    """One coarse cell's reduced model (romgen.hpp:23-45)."""
    cell: int = -1
    m: int = 0
    ktilde: int = 0
    shift: float = 0.0
    iface_ids: list = field(default_factory=list)      # ascending interface ids
    iface_offsets: list = field(default_factory=list)  # block offsets + total
    ladder_hat: list = field(default_factory=list)     # Lhat^1..Lhat^m (SPD)
    ladder: list = field(default_factory=list)         # L^1..L^m (SPD)
    g_proj: list = field(default_factory=list)         # per interface, length M
    q_proj: list = field(default_factory=list)
    # off-line diagnostics (not used on-line, not archived)
    V: np.ndarray | None = None
    Am: np.ndarray | None = None
    Bm: np.ndarray | None = None
    Sm: np.ndarray | None = None
    T: np.ndarray | None = None
    beta1: np.ndarray | None = None

    def block_offset(self, li: int) -> int:
        return self.iface_offsets[li]

    def block_size(self, li: int) -> int:
        return self.iface_offsets[li + 1] - self.iface_offsets[li]


@dataclass
class CoupledInterface:
    """One conjugated interface (msolver.hpp:16-25); cj = -1 single-sided."""
    part_iface: int = -1
    ci: int = -1
    cj: int = -1
    li: int = -1
    lj: int = -1
    size: int = 0
    S: np.ndarray | None = None
    mass: np.ndarray | None = None
    mass_form: np.ndarray | None = None
    g_proj: np.ndarray | None = None
    q_proj: np.ndarray | None = None


@dataclass
class CornerCopy:
    iface: int
    row: int
    mass: float


@dataclass
class CornerGroup:
    """Hanging copies of one removed corner node (msolver.hpp:28-36)."""
    parent: int = -1
    copies: list = field(default_factory=list)


@dataclass
class MultiscaleSystem:
    """Coupled ROM system (msolver.hpp:38-46)."""
    roms: list = field(default_factory=list)
    ifaces: list = field(default_factory=list)
    corners: list = field(default_factory=list)

    def total_reduced_io(self) -> int:  # msolver.cpp:8-12
        return sum(f.size for f in self.ifaces)

    def reduced_dof(self) -> int:  # msolver.cpp:14-18
        return sum(r.m * r.ktilde for r in self.roms)

    def flops_per_step(self) -> int:  # msolver.cpp:20-29
        fl = 0
        for r in self.roms:
            kt = r.ktilde
            fl += 2 * kt * kt + (r.m - 1) * 3 * 2 * kt * kt
        for f in self.ifaces:
            fl += 2 * f.size * f.size
        return fl


# ---------------------------------------------------------------------------
# flat (C ABI) form
# ---------------------------------------------------------------------------

class FlatSystem:
    """Plain arrays of ``msw_system_desc`` (include/mswave_b200.h)."""

    def __init__(self, cell_m, cell_ktilde, cell_iface_ptr, cell_iface_ids, cell_iface_offsets,
                 cell_ladder_off, ladders, iface_ci, iface_cj, iface_li, iface_lj, iface_size,
                 iface_mass=None):
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        self.cell_m = i32(cell_m)
        self.cell_ktilde = i32(cell_ktilde)
        self.cell_iface_ptr = i32(cell_iface_ptr)
        self.cell_iface_ids = i32(cell_iface_ids)
        self.cell_iface_offsets = i32(cell_iface_offsets)
        self.cell_ladder_off = np.ascontiguousarray(cell_ladder_off, dtype=np.int64)
        self.ladders = np.ascontiguousarray(ladders, dtype=np.float64)
        self.iface_ci = i32(iface_ci)
        self.iface_cj = i32(iface_cj)
        self.iface_li = i32(iface_li)
        self.iface_lj = i32(iface_lj)
        self.iface_size = i32(iface_size)
        self.iface_mass = None if iface_mass is None else np.ascontiguousarray(iface_mass, np.float64)
        self.iface_row_off = np.concatenate([[0], np.cumsum(self.iface_size, dtype=np.int64)])
        self.cell_u_off = np.concatenate(
            [[0], np.cumsum(self.cell_m.astype(np.int64) * self.cell_ktilde)])

    @property
    def n_cells(self) -> int:
        return int(self.cell_m.size)

    @property
    def n_ifaces(self) -> int:
        return int(self.iface_size.size)

    @property
    def total_io(self) -> int:
        return int(self.iface_row_off[-1])

    @property
    def total_u(self) -> int:
        return int(self.cell_u_off[-1])

    @property
    def n_flat(self) -> int:
        return self.total_io + int(np.sum((self.cell_m.astype(np.int64) - 1) * self.cell_ktilde))

    def dense_entries(self) -> int:
        kt = self.cell_ktilde.astype(np.int64)
        return int(np.sum((2 * self.cell_m.astype(np.int64) - 1) * kt * kt)
                   + np.sum(self.iface_size.astype(np.int64) ** 2))

    def ladder(self, c: int, k: int) -> np.ndarray:
        """L^{k+1} of cell c (column-major storage -> returned as a 2-D view)."""
        kt = int(self.cell_ktilde[c])
        o = int(self.cell_ladder_off[c]) + k * kt * kt
        return self.ladders[o:o + kt * kt].reshape(kt, kt).T

    def ladder_hat(self, c: int, k: int) -> np.ndarray:
        kt = int(self.cell_ktilde[c])
        m = int(self.cell_m[c])
        o = int(self.cell_ladder_off[c]) + (m + k) * kt * kt
        return self.ladders[o:o + kt * kt].reshape(kt, kt).T

    def desc(self) -> _ffi.SystemDesc:
        d = _ffi.SystemDesc()
        d.n_cells = self.n_cells
        d.n_ifaces = self.n_ifaces
        d.cell_m = ptr(self.cell_m, C.c_int32)
        d.cell_ktilde = ptr(self.cell_ktilde, C.c_int32)
        d.cell_iface_ptr = ptr(self.cell_iface_ptr, C.c_int32)
        d.cell_iface_ids = ptr(self.cell_iface_ids, C.c_int32)
        d.cell_iface_offsets = ptr(self.cell_iface_offsets, C.c_int32)
        d.cell_ladder_off = ptr(self.cell_ladder_off, C.c_int64)
        d.ladders = ptr(self.ladders)
        d.iface_ci = ptr(self.iface_ci, C.c_int32)
        d.iface_cj = ptr(self.iface_cj, C.c_int32)
        d.iface_li = ptr(self.iface_li, C.c_int32)
        d.iface_lj = ptr(self.iface_lj, C.c_int32)
        d.iface_size = ptr(self.iface_size, C.c_int32)
        d.iface_mass = ptr(self.iface_mass) if self.iface_mass is not None else None
        return d

    @staticmethod
    def from_system(sys: MultiscaleSystem, with_mass: bool = False) -> "FlatSystem":
        """Pack a reference-shaped MultiscaleSystem.  with_mass=True passes
        the interfaces' own ``mass`` (hand-built systems such as the
        reference's scalar_oscillator fixture); otherwise msw_create computes
        them from Lhat^1 exactly like assemble_system."""
        cm, ckt, cptr, cids, coff, loff, lad = [], [], [0], [], [], [], []
        off = 0
        for r in sys.roms:
            cm.append(r.m)
            ckt.append(r.ktilde)
            cids.extend(r.iface_ids)
            coff.extend(r.iface_offsets[:len(r.iface_ids)])
            cptr.append(len(cids))
            loff.append(off)
            for mat in list(r.ladder) + list(r.ladder_hat):
                a = np.asarray(mat, dtype=np.float64)
                lad.append(a.T.reshape(-1))  # column-major
                off += a.size
        mass = None
        if with_mass:
            mass = np.concatenate([np.asarray(f.mass, np.float64).T.reshape(-1) for f in sys.ifaces])
        return FlatSystem(cm, ckt, cptr, cids, coff, loff,
                          np.concatenate(lad) if lad else np.zeros(0),
                          [f.ci for f in sys.ifaces], [f.cj for f in sys.ifaces],
                          [f.li for f in sys.ifaces], [max(f.lj, -1) for f in sys.ifaces],
                          [f.size for f in sys.ifaces], mass)


@dataclass
class Receivers:
    """Flat receiver description: receiver r = sum over its terms of
    q_t . ubar_{iface_t} (msolver.cpp:405-411)."""
    rcv_ptr: np.ndarray
    term_iface: np.ndarray
    term_q: np.ndarray

    @property
    def R(self) -> int:
        return int(self.rcv_ptr.size - 1)

    @staticmethod
    def from_terms(terms: list) -> "Receivers":
        """terms: per receiver, a list of (iface, q vector) in ascending iface order."""
        ptr_, ifs, qs = [0], [], []
        for lst in terms:
            for f, q in lst:
                ifs.append(int(f))
                qs.append(np.asarray(q, dtype=np.float64).reshape(-1))
            ptr_.append(len(ifs))
        return Receivers(np.asarray(ptr_, np.int32), np.asarray(ifs, np.int32),
                         np.concatenate(qs) if qs else np.zeros(0))


# ---------------------------------------------------------------------------
# device stepper
# ---------------------------------------------------------------------------

class RomStepper:
    """Device-resident coupled ROM system (the C ABI msw_* handle)."""

    def __init__(self, flat: FlatSystem, device: int = 0):
        self.lib = _ffi.load()
        self.flat = flat
        h = C.c_void_p()
        d = flat.desc()
        _ffi.check(self.lib.msw_create(C.byref(d), device, C.byref(h)), self.lib)
        self.h = h
        self.S = 1
        self.R = 0

    @classmethod
    def from_archive(cls, directory: str, device: int = 0) -> "RomStepper":
        """msw_create_from_archive: load a reference ROM archive
        (rom_archive.cpp:110-190) straight onto the device, with the
        archive's own source / receiver as S = 1, R = 1."""
        from .archive import flat_from_archive, read_rom_archive
        self = cls.__new__(cls)
        self.lib = _ffi.load()
        self.flat = flat_from_archive(read_rom_archive(directory))
        h = C.c_void_p()
        _ffi.check(self.lib.msw_create_from_archive(directory.encode(), device, C.byref(h)), self.lib)
        self.h = h
        self.S = 1
        self.R = 1
        return self

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.msw_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, rc):
        _ffi.check(rc, self.lib)

    def info(self) -> dict:
        inf = _ffi.Info()
        self._c(self.lib.msw_get_info(self.h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in inf._fields_}

    def masses(self):
        n = int(np.sum(self.flat.iface_size.astype(np.int64) ** 2))
        mass = np.zeros(n)
        form = np.zeros(n)
        self._c(self.lib.msw_get_masses(self.h, ptr(mass), ptr(form)))
        return mass, form

    def estimate_dt(self, safety: float = 1.0) -> float:
        """msw_estimate_dt: estimate_dt (msolver.cpp:349-385) on the device."""
        out = C.c_double()
        self._c(self.lib.msw_estimate_dt(self.h, float(safety), C.byref(out)))
        return out.value

    def energy(self) -> np.ndarray:
        """msw_energy: energy (msolver.cpp:387-395) of the current state, per source."""
        out = np.zeros(self.S)
        self._c(self.lib.msw_energy(self.h, ptr(out)))
        return out

    def set_sources(self, g: np.ndarray):
        g = np.ascontiguousarray(g, dtype=np.float64)
        if g.ndim == 1:
            g = g[:, None]
        if g.shape[0] != self.flat.total_io:
            raise ConfigError("g_proj rows must equal sum_f M_f")
        self._c(self.lib.msw_set_sources(self.h, g.shape[1], ptr(g)))
        self.S = g.shape[1]

    def set_receivers(self, rc: Receivers):
        self._rc = rc
        self._c(self.lib.msw_set_receivers(self.h, rc.R, ptr(rc.rcv_ptr, C.c_int32),
                                           ptr(rc.term_iface, C.c_int32), ptr(rc.term_q)))
        self.R = rc.R

    def set_corners(self, grp_ptr, copy_iface, copy_row, copy_mass, iface_K, basis):
        a32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        self._corner = (a32(grp_ptr), a32(copy_iface), a32(copy_row),
                        np.ascontiguousarray(copy_mass, np.float64), a32(iface_K),
                        np.ascontiguousarray(basis, np.float64))
        gp, ci, cr, cm, ik, b = self._corner
        self._c(self.lib.msw_set_corners(self.h, gp.size - 1, ptr(gp, C.c_int32),
                                         ptr(ci, C.c_int32), ptr(cr, C.c_int32), ptr(cm),
                                         ptr(ik, C.c_int32), ptr(b)))

    def make_state(self, dt: float):
        self._c(self.lib.msw_make_state(self.h, float(dt)))

    def step(self, w):
        w = np.ascontiguousarray(np.atleast_1d(np.asarray(w, dtype=np.float64)))
        self._c(self.lib.msw_step(self.h, ptr(w), w.size))

    def corner_correct(self):
        self._c(self.lib.msw_corner_correct(self.h))

    def get_state(self) -> dict:
        S = self.S
        u_cur = np.zeros((self.flat.total_u, S))
        u_prev = np.zeros_like(u_cur)
        ub = np.zeros((self.flat.total_io, S))
        ubp = np.zeros_like(ub)
        t = C.c_double()
        si = C.c_int64()
        self._c(self.lib.msw_get_state(self.h, ptr(u_cur), ptr(u_prev), ptr(ub), ptr(ubp),
                                       C.byref(t), C.byref(si)))
        return dict(u_cur=u_cur, u_prev=u_prev, ubar_cur=ub, ubar_prev=ubp, t=t.value,
                    step_index=si.value)

    def set_state(self, u_cur, u_prev, ubar_cur, ubar_prev, t=0.0, step_index=0):
        arr = [np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, self.S))
               for a in (u_cur, u_prev, ubar_cur, ubar_prev)]
        self._c(self.lib.msw_set_state(self.h, *(ptr(a) for a in arr), float(t), int(step_index)))

    def run(self, steps: int, w: np.ndarray, corner: bool = False, traces_out=None,
            times_out=None):
        """run_simulation loop from the current state.  Returns
        (traces [steps+1, R, S], times [steps+1]).  traces_out / times_out may
        be preallocated (e.g. pinned) float64 arrays of those shapes."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        stride = 1 if w.ndim == 1 else w.shape[1]
        if w.shape[0] < steps:
            raise ConfigError("not enough wavelet samples")
        traces = traces_out if traces_out is not None else np.zeros((steps + 1, self.R, self.S))
        times = times_out if times_out is not None else np.zeros(steps + 1)
        if traces.size != (steps + 1) * self.R * self.S or times.size != steps + 1:
            raise ConfigError("output buffers have the wrong size")
        bad = C.c_int64()
        rc = self.lib.msw_run(self.h, int(steps), ptr(w), stride, int(bool(corner)),
                              ptr(traces), ptr(times), C.byref(bad))
        self._c(rc)
        return traces, times

    def run_device(self, steps: int, w_dev_ptr: int, w_stride: int, traces_dev_ptr: int,
                   stream: int | None = None, corner: bool = False):
        self._c(self.lib.msw_run_device(self.h, int(steps), C.c_void_p(w_dev_ptr), int(w_stride),
                                        int(bool(corner)), C.c_void_p(traces_dev_ptr),
                                        C.c_void_p(stream or 0)))

    def prepare(self, corner: bool = False):
        """Instantiate the step graph now (keeps setup out of timed regions)."""
        self._c(self.lib.msw_prepare(self.h, int(bool(corner))))

    def check_instability(self) -> int:
        bad = C.c_int64()
        rc = self.lib.msw_check_instability(self.h, C.byref(bad))
        if rc not in (_ffi.MSW_OK, _ffi.MSW_NUMERICAL_ERROR):
            self._c(rc)
        return bad.value

    def time_kernels(self, reps: int = 20):
        """Average per-launch ms of (K1 cell kernel, K2 interface kernel),
        each timed alone with CUDA events.  Scrambles the state."""
        ms = np.zeros(2)
        self._c(self.lib.msw_time_kernels(self.h, int(reps), ptr(ms)))
        return float(ms[0]), float(ms[1])

    def last_launches(self) -> int:
        n = C.c_int64()
        self._c(self.lib.msw_last_launch_count(self.h, C.byref(n)))
        return n.value


def system_sources(sys: MultiscaleSystem) -> np.ndarray:
    """The system's single projected source g~ (CoupledInterface::g_proj) as
    a [sum_f M_f, 1] array."""
    return np.concatenate([np.asarray(f.g_proj, np.float64).reshape(-1) for f in sys.ifaces])[:, None]


def system_receiver(sys: MultiscaleSystem) -> Receivers:
    """The system's single receiver sum_f q~_f . ubar_f (msolver.cpp:405-411);
    interfaces whose q~ is identically zero contribute exact zeros and are
    omitted."""
    terms = [(f, np.asarray(cf.q_proj, np.float64)) for f, cf in enumerate(sys.ifaces)
             if cf.q_proj is not None and np.any(np.asarray(cf.q_proj) != 0.0)]
    return Receivers.from_terms([terms])
