"""Fine-grid companion: medium, pencil numbering, sources/receivers and the
device leapfrog handle (msw_fine_*).

Mirrors proj/include/mswave/fine_grid.hpp and reference.hpp:
  GridMedium            fine_grid.hpp:14-23
  SparsePencil.node_of  fine_grid.cpp:29-36 (row-major over interior dims)
  make_source           fine_grid.cpp:119-165 (Point, UnitImpulse, Taper)
  set_receiver          fine_grid.cpp:167-174
  fine_leapfrog         reference.cpp:49-80   (device kernel)
  fine_cfl              reference.cpp:24-47   (device power iteration)

Two kinds of device handle: FineGrid(medium) applies the stencil matrix-free
from sigma / rho (the throughput path); FineGrid.from_pencil(pencil) takes any
assembled SparsePencil -- A as Eigen stores it (CSC), e.g. the corner-modified
pencil with hanging copies -- and sums rows in the reference's column order.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _ffi
from ._ffi import ConfigError, ptr


@dataclass
class GridMedium:
    dims: list
    h: float = 1.0
    sigma: np.ndarray | None = None
    rho: np.ndarray | None = None

    def ndim(self) -> int:
        return len(self.dims)

    def node_count(self) -> int:
        return int(np.prod(self.dims))

    def node_id(self, c) -> int:  # fine_grid.cpp:13-17
        i = 0
        for a in range(self.ndim()):
            i = i * self.dims[a] + int(c[a])
        return i


def make_uniform_medium(dims, h, sigma_value, rho_value=1.0) -> GridMedium:
    n = int(np.prod(dims))
    return GridMedium(list(dims), float(h), np.full(n, float(sigma_value)), np.full(n, float(rho_value)))


def interior_size(dims) -> int:
    return int(np.prod([d - 2 for d in dims]))


def node_of(dims, c) -> int:
    """Interior row of a full-grid coordinate, -1 outside (fine_grid.cpp:29-36)."""
    i = 0
    for a in range(len(dims)):
        if c[a] < 1 or c[a] > dims[a] - 2:
            return -1
        i = i * (dims[a] - 2) + (int(c[a]) - 1)
    return i


def interior_coords(dims) -> np.ndarray:
    """coords of every interior row (SparsePencil::coords, unused axes 0)."""
    nd = len(dims)
    idims = [d - 2 for d in dims]
    grids = np.meshgrid(*[np.arange(1, d - 1) for d in dims], indexing="ij")
    out = np.zeros((interior_size(dims), 3), dtype=np.int64)
    for a in range(nd):
        out[:, a] = grids[a].reshape(-1)
    return out


@dataclass
class SparseVec:
    """A sparse source/receiver vector over interior rows (ascending rows)."""
    rows: np.ndarray
    vals: np.ndarray


def make_source(dims, location, kind: str = "point", rho: np.ndarray | None = None,
                taper_axis: int = 0, taper_halfwidth: float = 3.0) -> SparseVec:
    """fine_grid.cpp:119-165.  rho: full-grid density (UnitImpulse only)."""
    k = node_of(dims, location)
    if k < 0:
        raise ConfigError("source location outside the interior grid")
    if kind == "point":
        return SparseVec(np.array([k], np.int64), np.array([1.0]))
    if kind == "unit_impulse":
        gid = 0
        for a in range(len(dims)):
            gid = gid * dims[a] + int(location[a])
        return SparseVec(np.array([k], np.int64), np.array([1.0 / rho[gid]]))
    if kind == "taper":
        nd = len(dims)
        if taper_axis < 0 or taper_axis >= nd:
            raise ConfigError("taper axis out of range")
        hw = taper_halfwidth
        reach = int(math.ceil(3.0 * hw))
        coords = interior_coords(dims)
        rows, vals = [], []
        total = 0.0
        for row in range(coords.shape[0]):
            c = coords[row]
            if c[taper_axis] != location[taper_axis]:
                continue
            d2 = 0.0
            close = True
            for a in range(nd):
                if a == taper_axis:
                    continue
                d = int(c[a]) - int(location[a])
                if abs(d) > reach:
                    close = False
                    break
                d2 += float(d) * d
            if not close:
                continue
            w = math.exp(-0.5 * d2 / (hw * hw))
            rows.append(row)
            vals.append(w)
            total += w
        if total <= 0.0:
            raise ConfigError("taper source has empty support")
        return SparseVec(np.array(rows, np.int64), np.array(vals) / total)
    raise ConfigError(f"unknown source kind {kind}")


def set_receiver(dims, location) -> SparseVec:
    k = node_of(dims, location)
    if k < 0:
        raise ConfigError("receiver location outside the interior grid")
    return SparseVec(np.array([k], np.int64), np.array([1.0]))


def _csr(vecs: list):
    ptr_ = [0]
    rows, vals = [], []
    for v in vecs:
        rows.append(np.asarray(v.rows, np.int64))
        vals.append(np.asarray(v.vals, np.float64))
        ptr_.append(ptr_[-1] + len(v.rows))
    return (np.asarray(ptr_, np.int32),
            np.ascontiguousarray(np.concatenate(rows) if rows else np.zeros(0, np.int64)),
            np.ascontiguousarray(np.concatenate(vals) if vals else np.zeros(0)))


def gershgorin_lambda(medium: GridMedium) -> float:
    """Upper bound of lambda_max(B^-1 (-A)) (reference.cpp:11-20) computed
    from sigma/rho: max_i (|diag_i| + sum_j |a_ij|) / B_i = 2|diag_i|/B_i
    minus the Dirichlet edges; here the bound 2*sum(edges)/rho is used."""
    nd = medium.ndim()
    sig = medium.sigma.reshape(medium.dims)
    rho = medium.rho.reshape(medium.dims)
    inner = tuple(slice(1, d - 1) for d in medium.dims)
    tot = np.zeros([d - 2 for d in medium.dims])
    for a in range(nd):
        for sh in (-1, 1):
            nb = list(inner)
            nb[a] = slice(1 + sh, medium.dims[a] - 1 + sh)
            tot += 0.5 * (sig[inner] + sig[tuple(nb)])
    return float(np.max(2.0 * tot / (medium.h ** 2) / rho[inner]))


class FineGrid:
    """Device-resident fine-grid leapfrog (msw_fine_* handle)."""

    def __init__(self, medium: GridMedium, device: int = 0):
        self.lib = _ffi.load()
        self.medium = medium
        self.dims = np.asarray(medium.dims, np.int32)
        sig = np.ascontiguousarray(medium.sigma, np.float64)
        rho = np.ascontiguousarray(medium.rho, np.float64)
        h = C.c_void_p()
        _ffi.check(self.lib.msw_fine_create(len(medium.dims), ptr(self.dims, C.c_int32),
                                            float(medium.h), ptr(sig), ptr(rho), device,
                                            C.byref(h)), self.lib)
        self.h = h

    @classmethod
    def from_pencil(cls, pencil, device: int = 0) -> "FineGrid":
        """Device handle of an assembled pencil (offline.partition.Pencil or
        anything with a scipy CSC ``A`` and a diagonal ``B``):
        msw_fine_create_csc."""
        self = cls.__new__(cls)
        self.lib = _ffi.load()
        self.medium = None
        A = pencil.A.tocsc()
        A.sort_indices()
        n = A.shape[0]
        outer = np.ascontiguousarray(A.indptr, np.int32)
        inner = np.ascontiguousarray(A.indices, np.int32)
        vals = np.ascontiguousarray(A.data, np.float64)
        B = np.ascontiguousarray(pencil.B, np.float64)
        h = C.c_void_p()
        _ffi.check(self.lib.msw_fine_create_csc(n, ptr(outer, C.c_int32), ptr(inner, C.c_int32), ptr(vals),
                                                ptr(B), device, C.byref(h)), self.lib)
        self.h = h
        self.dims = None
        return self

    def cfl(self) -> float:
        """fine_cfl (reference.cpp:24-47) on the device: 2 / sqrt(lambda_max)."""
        out = C.c_double()
        _ffi.check(self.lib.msw_fine_cfl(self.h, C.byref(out)), self.lib)
        return out.value

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.msw_fine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        n = C.c_int64()
        _ffi.check(self.lib.msw_fine_size(self.h, C.byref(n)), self.lib)
        return n.value

    def leapfrog(self, sources: list, receivers: list, dt: float, steps: int, w: np.ndarray):
        """fine_leapfrog for S sources / R receivers; w [steps] or [steps, S]
        sampled at t_s = s*dt.  Returns traces [steps+1, R, S]."""
        S, R = len(sources), len(receivers)
        sp, sr, sv = _csr(sources)
        rp, rr, rv = _csr(receivers)
        w = np.ascontiguousarray(w, np.float64)
        stride = 1 if w.ndim == 1 else w.shape[1]
        traces = np.zeros((steps + 1, R, S))
        bad = C.c_int64()
        rc = self.lib.msw_fine_leapfrog(self.h, S, ptr(sp, C.c_int32), ptr(sr, C.c_int64), ptr(sv),
                                        R, ptr(rp, C.c_int32), ptr(rr, C.c_int64), ptr(rv),
                                        float(dt), int(steps), ptr(w), stride, ptr(traces),
                                        C.byref(bad))
        _ffi.check(rc, self.lib)
        return traces

    def leapfrog_device(self, sources: list, receivers: list, dt: float, steps: int,
                        w_dev_ptr: int, w_stride: int, traces_dev_ptr: int, reset: bool = True,
                        stream: int | None = None):
        S, R = len(sources), len(receivers)
        self._io = (_csr(sources), _csr(receivers))
        (sp, sr, sv), (rp, rr, rv) = self._io
        _ffi.check(self.lib.msw_fine_leapfrog_device(
            self.h, S, ptr(sp, C.c_int32), ptr(sr, C.c_int64), ptr(sv), R, ptr(rp, C.c_int32),
            ptr(rr, C.c_int64), ptr(rv), float(dt), int(steps), C.c_void_p(w_dev_ptr),
            int(w_stride), C.c_void_p(traces_dev_ptr), int(bool(reset)), C.c_void_p(stream or 0)),
            self.lib)

    def check_instability(self) -> int:
        bad = C.c_int64()
        rc = self.lib.msw_fine_check_instability(self.h, C.byref(bad))
        if rc not in (_ffi.MSW_OK, _ffi.MSW_NUMERICAL_ERROR):
            _ffi.check(rc, self.lib)
        return bad.value
