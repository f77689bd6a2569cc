"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/liboracle.so, the CPU
restatement of the reference's on-line stepper and fine leapfrog (see
oracle/oracle.cpp for the file:line map).  Same method surface as the
product's RomStepper / FineGrid so parity tests read symmetrically."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1604_06750_b200 import _ffi
from paper_1604_06750_b200._ffi import ConfigError, NumericalError, ptr
from paper_1604_06750_b200.rom import FlatSystem, Receivers

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
i32p, i64p, f64p = _ffi.i32p, _ffi.i64p, _ffi.f64p

_PROTOS = {
    "oracle_last_error": (C.c_char_p, []),
    "oracle_create": (C.c_int, [C.POINTER(_ffi.SystemDesc), C.POINTER(C.c_void_p)]),
    "oracle_destroy": (None, [C.c_void_p]),
    "oracle_get_masses": (C.c_int, [C.c_void_p, f64p, f64p]),
    "oracle_set_sources": (C.c_int, [C.c_void_p, C.c_int, f64p]),
    "oracle_set_receivers": (C.c_int, [C.c_void_p, C.c_int, i32p, i32p, f64p]),
    "oracle_set_corners": (C.c_int, [C.c_void_p, C.c_int, i32p, i32p, i32p, f64p, i32p, f64p]),
    "oracle_make_state": (C.c_int, [C.c_void_p, C.c_double]),
    "oracle_step": (C.c_int, [C.c_void_p, f64p, C.c_int]),
    "oracle_corner_correct": (C.c_int, [C.c_void_p]),
    "oracle_get_state": (C.c_int, [C.c_void_p, f64p, f64p, f64p, f64p, f64p, i64p]),
    "oracle_set_state": (C.c_int, [C.c_void_p, f64p, f64p, f64p, f64p, C.c_double, C.c_int64]),
    "oracle_run": (C.c_int, [C.c_void_p, C.c_int64, f64p, C.c_int, C.c_int, f64p, f64p, i64p,
                             C.c_int]),
    "oracle_estimate_dt": (C.c_int, [C.c_void_p, C.c_double, f64p]),
    "oracle_energy": (C.c_int, [C.c_void_p, f64p]),
    "oracle_wavelet": (C.c_double, [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]),
    "oracle_fine_create": (C.c_int, [C.c_int, i32p, C.c_double, f64p, f64p, C.POINTER(C.c_void_p)]),
    "oracle_fine_create_csr": (C.c_int, [C.c_int64, i64p, i64p, f64p, f64p, C.POINTER(C.c_void_p)]),
    "oracle_fine_destroy": (None, [C.c_void_p]),
    "oracle_fine_size": (C.c_int64, [C.c_void_p]),
    "oracle_fine_nnz": (C.c_int64, [C.c_void_p]),
    "oracle_fine_export": (C.c_int, [C.c_void_p, i64p, i64p, f64p, f64p]),
    "oracle_fine_cfl": (C.c_int, [C.c_void_p, f64p]),
    "oracle_fine_leapfrog": (C.c_int, [C.c_void_p, C.c_int, i32p, i64p, f64p, C.c_int, i32p, i64p,
                                       f64p, C.c_double, C.c_int64, f64p, C.c_int, f64p, i64p,
                                       C.c_int]),
    "oracle_compare_traces": (C.c_int, [f64p, f64p, C.c_int64, f64p, f64p, C.c_int64, f64p, f64p]),
}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        for k, (r, a) in _PROTOS.items():
            f = getattr(lib, k)
            f.restype = r
            f.argtypes = a
        _lib = lib
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = load().oracle_last_error().decode()
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise NumericalError(msg)
    raise RuntimeError(msg)


class OracleStepper:
    """CPU restatement of assemble_system/make_state/step/run_simulation."""

    def __init__(self, flat: FlatSystem):
        self.lib = load()
        self.flat = flat
        h = C.c_void_p()
        d = flat.desc()
        _check(self.lib.oracle_create(C.byref(d), C.byref(h)))
        self.h = h
        self.S = 1
        self.R = 0

    def __del__(self):
        try:
            if self.h is not None and self.h.value:
                self.lib.oracle_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def masses(self):
        n = int(np.sum(self.flat.iface_size.astype(np.int64) ** 2))
        mass, form = np.zeros(n), np.zeros(n)
        _check(self.lib.oracle_get_masses(self.h, ptr(mass), ptr(form)))
        return mass, form

    def set_sources(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        if g.ndim == 1:
            g = g[:, None]
        _check(self.lib.oracle_set_sources(self.h, g.shape[1], ptr(g)))
        self.S = g.shape[1]

    def set_receivers(self, rc: Receivers):
        self._rc = rc
        _check(self.lib.oracle_set_receivers(self.h, rc.R, ptr(rc.rcv_ptr, C.c_int32),
                                             ptr(rc.term_iface, C.c_int32), ptr(rc.term_q)))
        self.R = rc.R

    def set_corners(self, grp_ptr, copy_iface, copy_row, copy_mass, iface_K, basis):
        a32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        self._corner = (a32(grp_ptr), a32(copy_iface), a32(copy_row),
                        np.ascontiguousarray(copy_mass, np.float64), a32(iface_K),
                        np.ascontiguousarray(basis, np.float64))
        gp, ci, cr, cm, ik, b = self._corner
        _check(self.lib.oracle_set_corners(self.h, gp.size - 1, ptr(gp, C.c_int32), ptr(ci, C.c_int32),
                                           ptr(cr, C.c_int32), ptr(cm), ptr(ik, C.c_int32), ptr(b)))

    def make_state(self, dt):
        _check(self.lib.oracle_make_state(self.h, float(dt)))

    def step(self, w):
        w = np.ascontiguousarray(np.atleast_1d(np.asarray(w, dtype=np.float64)))
        _check(self.lib.oracle_step(self.h, ptr(w), w.size))

    def corner_correct(self):
        _check(self.lib.oracle_corner_correct(self.h))

    def get_state(self):
        S = self.S
        u_cur = np.zeros((self.flat.total_u, S))
        u_prev = np.zeros_like(u_cur)
        ub = np.zeros((self.flat.total_io, S))
        ubp = np.zeros_like(ub)
        t = C.c_double()
        si = C.c_int64()
        _check(self.lib.oracle_get_state(self.h, ptr(u_cur), ptr(u_prev), ptr(ub), ptr(ubp),
                                         C.byref(t), C.byref(si)))
        return dict(u_cur=u_cur, u_prev=u_prev, ubar_cur=ub, ubar_prev=ubp, t=t.value,
                    step_index=si.value)

    def set_state(self, u_cur, u_prev, ubar_cur, ubar_prev, t=0.0, step_index=0):
        arr = [np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, self.S))
               for a in (u_cur, u_prev, ubar_cur, ubar_prev)]
        _check(self.lib.oracle_set_state(self.h, *(ptr(a) for a in arr), float(t), int(step_index)))

    def run(self, steps, w, corner=False, threads=1):
        w = np.ascontiguousarray(w, dtype=np.float64)
        stride = 1 if w.ndim == 1 else w.shape[1]
        traces = np.zeros((steps + 1, self.R, self.S))
        times = np.zeros(steps + 1)
        bad = C.c_int64()
        _check(self.lib.oracle_run(self.h, int(steps), ptr(w), stride, int(bool(corner)),
                                   ptr(traces), ptr(times), C.byref(bad), int(threads)))
        return traces, times

    def estimate_dt(self, safety=1.0):
        out = C.c_double()
        _check(self.lib.oracle_estimate_dt(self.h, float(safety), C.byref(out)))
        return out.value

    def energy(self):
        e = np.zeros(self.S)
        _check(self.lib.oracle_energy(self.h, ptr(e)))
        return e


class OracleFine:
    def __init__(self, medium=None, csr=None):
        self.lib = load()
        h = C.c_void_p()
        if medium is not None:
            dims = np.asarray(medium.dims, np.int32)
            _check(self.lib.oracle_fine_create(len(medium.dims), ptr(dims, C.c_int32), float(medium.h),
                                               ptr(np.ascontiguousarray(medium.sigma, np.float64)),
                                               ptr(np.ascontiguousarray(medium.rho, np.float64)),
                                               C.byref(h)))
        else:
            n, p, c, v, B = csr
            self._keep = [np.ascontiguousarray(x) for x in (p, c, v, B)]
            p, c, v, B = self._keep
            _check(self.lib.oracle_fine_create_csr(int(n), ptr(p, C.c_int64), ptr(c, C.c_int64),
                                                   ptr(v), ptr(B), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h is not None and self.h.value:
                self.lib.oracle_fine_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def n(self):
        return self.lib.oracle_fine_size(self.h)

    def pencil(self):
        n = self.n
        nnz = self.lib.oracle_fine_nnz(self.h)
        p = np.zeros(n + 1, np.int64)
        c = np.zeros(nnz, np.int64)
        v = np.zeros(nnz)
        B = np.zeros(n)
        _check(self.lib.oracle_fine_export(self.h, ptr(p, C.c_int64), ptr(c, C.c_int64), ptr(v), ptr(B)))
        return p, c, v, B

    def cfl(self):
        out = C.c_double()
        _check(self.lib.oracle_fine_cfl(self.h, C.byref(out)))
        return out.value

    def leapfrog(self, sources, receivers, dt, steps, w, threads=1):
        from paper_1604_06750_b200.fine import _csr
        S, R = len(sources), len(receivers)
        sp, sr, sv = _csr(sources)
        rp, rr, rv = _csr(receivers)
        w = np.ascontiguousarray(w, np.float64)
        stride = 1 if w.ndim == 1 else w.shape[1]
        traces = np.zeros((steps + 1, R, S))
        bad = C.c_int64()
        _check(self.lib.oracle_fine_leapfrog(self.h, S, ptr(sp, C.c_int32), ptr(sr, C.c_int64), ptr(sv),
                                             R, ptr(rp, C.c_int32), ptr(rr, C.c_int64), ptr(rv),
                                             float(dt), int(steps), ptr(w), stride, ptr(traces),
                                             C.byref(bad), int(threads)))
        return traces


def wavelet(kind, omega_cut, width, delay, t):
    return load().oracle_wavelet(kind, omega_cut, width, delay, t)


def compare_traces(at, av, bt, bv):
    at, av, bt, bv = (np.ascontiguousarray(x, np.float64) for x in (at, av, bt, bv))
    mx, rl = C.c_double(), C.c_double()
    _check(load().oracle_compare_traces(ptr(at), ptr(av), at.size, ptr(bt), ptr(bv), bt.size,
                                        C.byref(mx), C.byref(rl)))
    return mx.value, rl.value
