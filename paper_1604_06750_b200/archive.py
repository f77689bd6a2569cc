"""ROM archive: the off-line artifact the on-line stepper loads
(rom_archive.hpp:12-26, rom_archive.cpp:65-190), and the multi-source /
multi-receiver projection onto it (romgen.cpp:359-363, 446-455).

On-disk format (identical bytes to the reference writer):
  manifest.json      {"format": "mswave-rom-archive", "version": 1,
                      "num_cells", "num_interfaces", "omega_max", "epsilon",
                      "m", "max_basis_per_interface",
                      "cells": [{"file", "ktilde", "m", "interfaces"}]}
  cell_%04d.bin      magic "MSWROM1\\0"; u64 cell, m, ktilde, n_ifaces;
                     f64 shift; per interface: u64 id, mat S_f, u64 M,
                     f64[M] g_proj, f64[M] q_proj; then mat Lhat^1..m,
                     mat L^1..m.   mat = u64 rows, u64 cols, f64 col-major.
All integers are 64-bit little endian, all floats IEEE binary64 little endian.

The archive stores each interface basis S_f, so sources and receivers other
than the one the ROMs were built with are projected here
(g~_f = S_f^T g|_f, romgen.cpp:359-363): ``project_sources`` /
``project_receivers`` batch S of them for the on-line stepper.
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass

import numpy as np

from ._ffi import ConfigError
from .offline.romgen import BoundaryBasis, RomOptions
from .rom import Receivers, SubdomainROM

MAGIC = b"MSWROM1\x00"


def _cell_filename(cell: int) -> str:
    return "cell_%04d.bin" % cell


def _put_mat(buf: list, m: np.ndarray) -> None:
    m = np.asarray(m, dtype=np.float64)
    if m.ndim == 1:
        m = m.reshape(-1, 1)
    buf.append(struct.pack("<QQ", m.shape[0], m.shape[1]))
    buf.append(np.asfortranarray(m).tobytes(order="F"))


@dataclass
class RomArchive:
    """rom_archive.hpp:19-23."""
    roms: list
    basis: BoundaryBasis
    opt: RomOptions


def write_rom_archive(directory: str, roms: list, basis: BoundaryBasis, opt: RomOptions) -> None:
    """rom_archive.cpp:65-108."""
    os.makedirs(directory, exist_ok=True)
    cells = []
    for rom in roms:
        cells.append({"file": _cell_filename(rom.cell), "ktilde": int(rom.ktilde), "m": int(rom.m),
                      "interfaces": [int(f) for f in rom.iface_ids]})
        buf = [MAGIC, struct.pack("<QQQQ", rom.cell, rom.m, rom.ktilde, len(rom.iface_ids)),
               struct.pack("<d", float(rom.shift))]
        for li, f in enumerate(rom.iface_ids):
            buf.append(struct.pack("<Q", int(f)))
            _put_mat(buf, basis.S[f])
            g = np.asarray(rom.g_proj[li], dtype=np.float64).reshape(-1)
            q = np.asarray(rom.q_proj[li], dtype=np.float64).reshape(-1)
            buf.append(struct.pack("<Q", g.size))
            buf.append(g.tobytes())
            buf.append(q.tobytes())
        for m in rom.ladder_hat:
            _put_mat(buf, m)
        for m in rom.ladder:
            _put_mat(buf, m)
        with open(os.path.join(directory, _cell_filename(rom.cell)), "wb") as fh:
            fh.write(b"".join(buf))
    manifest = {"format": "mswave-rom-archive", "version": 1, "num_cells": len(roms),
                "num_interfaces": len(basis.S), "omega_max": float(basis.omega_max),
                "epsilon": float(basis.epsilon), "m": int(opt.m),
                "max_basis_per_interface": int(opt.max_basis_per_interface), "cells": cells}
    with open(os.path.join(directory, "manifest.json"), "w") as fh:
        fh.write(json.dumps(manifest, indent=2) + "\n")


class _Reader:
    def __init__(self, data: bytes, path: str):
        self.data, self.pos, self.path = data, 0, path

    def u64(self) -> int:
        if self.pos + 8 > len(self.data):
            raise ConfigError("truncated ROM container")
        v = struct.unpack_from("<Q", self.data, self.pos)[0]
        self.pos += 8
        return v

    def doubles(self, n: int) -> np.ndarray:
        if self.pos + 8 * n > len(self.data):
            raise ConfigError("truncated ROM container payload")
        v = np.frombuffer(self.data, dtype="<f8", count=n, offset=self.pos).astype(np.float64)
        self.pos += 8 * n
        return v

    def mat(self) -> np.ndarray:
        rows, cols = self.u64(), self.u64()
        if rows > (1 << 24) or cols > (1 << 24):
            raise ConfigError("implausible matrix dimensions in ROM container")
        return self.doubles(rows * cols).reshape((rows, cols), order="F")


def read_rom_archive(directory: str) -> RomArchive:
    """rom_archive.cpp:110-190 (same checks, same messages)."""
    mpath = os.path.join(directory, "manifest.json")
    if not os.path.exists(mpath):
        raise ConfigError("missing manifest.json in " + directory)
    with open(mpath) as fh:
        manifest = json.load(fh)
    if manifest.get("format", "") != "mswave-rom-archive":
        raise ConfigError("not a ROM archive: " + directory)
    opt = RomOptions(m=int(manifest["m"]), omega_max=float(manifest["omega_max"]),
                     epsilon_rel=float(manifest["epsilon"]),
                     max_basis_per_interface=int(manifest.get("max_basis_per_interface", 0)))
    nf = int(manifest["num_interfaces"])
    basis = BoundaryBasis(omega_max=opt.omega_max, epsilon=opt.epsilon_rel, S=[None] * nf,
                          kept_eigs=[np.zeros(0)] * nf, tail=[0.0] * nf)
    roms = []
    for c in manifest["cells"]:
        path = os.path.join(directory, c["file"])
        if not os.path.exists(path):
            raise ConfigError("missing ROM container: " + path)
        with open(path, "rb") as fh:
            data = fh.read()
        if data[:8] != MAGIC:
            raise ConfigError("bad magic in ROM container: " + path)
        rd = _Reader(data, path)
        rd.pos = 8
        rom = SubdomainROM(cell=rd.u64(), m=rd.u64(), ktilde=rd.u64())
        nif = rd.u64()
        rom.shift = float(rd.doubles(1)[0])
        rom.iface_offsets = [0]
        for _ in range(nif):
            fid = rd.u64()
            rom.iface_ids.append(fid)
            S = rd.mat()
            glen = rd.u64()
            g, q = rd.doubles(glen), rd.doubles(glen)
            if S.shape[1] != glen:
                raise ConfigError("interface basis / projected I/O size mismatch in " + path)
            if fid >= nf:
                raise ConfigError("interface id out of range in " + path)
            if basis.S[fid] is None:
                basis.S[fid] = S
            elif basis.S[fid].shape != S.shape or basis.S[fid].tobytes(order="F") != S.tobytes(order="F"):
                raise ConfigError("mismatched interface bases between neighbor cells (interface %d)" % fid)
            rom.g_proj.append(g)
            rom.q_proj.append(q)
            rom.iface_offsets.append(rom.iface_offsets[-1] + glen)
        rom.ladder_hat = [rd.mat() for _ in range(rom.m)]
        rom.ladder = [rd.mat() for _ in range(rom.m)]
        if rom.iface_offsets[-1] != rom.ktilde:
            raise ConfigError("inconsistent ktilde in " + path)
        roms.append(rom)
    roms.sort(key=lambda r: r.cell)
    return RomArchive(roms, basis, opt)


def _support_on_iface(nodes: np.ndarray, vec) -> np.ndarray:
    """values of a (dense or (rows, vals) sparse) fine vector on an interface's
    sorted node list."""
    if isinstance(vec, tuple):
        rows, vals = (np.asarray(vec[0], np.int64), np.asarray(vec[1], np.float64))
        out = np.zeros(nodes.size)
        pos = np.searchsorted(nodes, rows)
        ok = (pos < nodes.size) & (nodes[np.minimum(pos, nodes.size - 1)] == rows)
        np.add.at(out, pos[ok], vals[ok])
        return out
    return np.asarray(vec, np.float64)[nodes]


def _check_skeleton(part, vec, what: str) -> None:
    """romgen.cpp:463-475: support off the partition skeleton is an error."""
    on = np.zeros(part.n_nodes, bool)
    on[part.skeleton] = True
    if isinstance(vec, tuple):
        rows = np.asarray(vec[0], np.int64)[np.asarray(vec[1]) != 0.0]
    else:
        rows = np.nonzero(np.asarray(vec))[0]
    bad = rows[~on[rows]]
    if bad.size:
        raise ConfigError(what + " has support off the partition skeleton at nodes: " +
                          " ".join(str(int(k)) for k in bad))


def project_sources(part, basis: BoundaryBasis, sources: list) -> np.ndarray:
    """S sources (dense fine vectors or (rows, values) pairs on the modified
    pencil) -> g~ [sum_f M_f, S], interfaces in basis order, each
    g~_f = S_f^T g|_f (romgen.cpp:359-363, 446-455)."""
    sizes = [basis.S[f].shape[1] for f in range(len(basis.S))]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    G = np.zeros((int(off[-1]), len(sources)))
    for s, vec in enumerate(sources):
        _check_skeleton(part, vec, "source")
        for f, I in enumerate(part.interfaces):
            gr = _support_on_iface(np.asarray(I.nodes, np.int64), vec)
            if np.any(gr != 0.0):
                G[off[f]:off[f + 1], s] = basis.S[f].T @ gr
    return G


def project_receivers(part, basis: BoundaryBasis, receivers: list) -> Receivers:
    """R receivers -> per receiver the interfaces its support touches with
    q~_f = S_f^T q|_f; the trace is sum_f q~_f . ubar_f (msolver.cpp:405-411)."""
    terms = []
    for vec in receivers:
        _check_skeleton(part, vec, "receiver")
        lst = []
        for f, I in enumerate(part.interfaces):
            qr = _support_on_iface(np.asarray(I.nodes, np.int64), vec)
            if np.any(qr != 0.0):
                lst.append((f, basis.S[f].T @ qr))
        terms.append(lst)
    return Receivers.from_terms(terms)


def flat_from_archive(ar: RomArchive):
    """msw_system_desc arrays straight from an archive, no partition: the
    interface topology msw_create_from_archive derives (an interface's first
    listing cell is ci, the second cj), masses left to msw_create."""
    from .rom import FlatSystem
    nf = len(ar.basis.S)
    ci, cj, li, lj = [-1] * nf, [-1] * nf, [-1] * nf, [-1] * nf
    cm, ckt, cptr, cids, coff, loff, lad = [], [], [0], [], [], [], []
    off = 0
    for c, r in enumerate(ar.roms):
        if r.cell != c:
            raise ConfigError("ROM archive cells are not numbered 0..n-1")
        cm.append(r.m)
        ckt.append(r.ktilde)
        for l, f in enumerate(r.iface_ids):
            if ci[f] < 0:
                ci[f], li[f] = c, l
            elif cj[f] < 0:
                cj[f], lj[f] = c, l
            else:
                raise ConfigError("interface %d listed by more than two cells" % f)
        cids.extend(r.iface_ids)
        coff.extend(r.iface_offsets[:len(r.iface_ids)])
        cptr.append(len(cids))
        loff.append(off)
        for mat in list(r.ladder) + list(r.ladder_hat):
            lad.append(np.asarray(mat, np.float64).T.reshape(-1))
            off += mat.size
    sizes = [ar.basis.S[f].shape[1] for f in range(nf)]
    return FlatSystem(cm, ckt, cptr, cids, coff, loff, np.concatenate(lad), ci, cj, li, lj, sizes)


def archive_io(ar: RomArchive):
    """The archive's own projected source (g~, [sum_f M_f, 1]) and receiver."""
    flat = flat_from_archive(ar)
    g = np.zeros((flat.total_io, 1))
    terms = []
    for f in range(flat.n_ifaces):
        c, l = int(flat.iface_ci[f]), int(flat.iface_li[f])
        g[flat.iface_row_off[f]:flat.iface_row_off[f + 1], 0] = ar.roms[c].g_proj[l]
        q = ar.roms[c].q_proj[l]
        if np.any(q != 0.0):
            terms.append((f, q))
    return g, Receivers.from_terms([terms])


def system_from_archive(part, ar: RomArchive, B_diag):
    """cmd_simulate's on-line load (cli_commands.cpp:111-116): archive +
    re-staged partition -> assemble_system (msolver.cpp:31-106)."""
    from .offline.romgen import assemble_system
    if len(ar.roms) != part.num_cells():
        raise ConfigError("ROM archive cell count does not match the partition")
    return assemble_system(part, ar.basis, ar.roms, B_diag)
