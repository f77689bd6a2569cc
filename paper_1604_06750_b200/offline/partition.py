"""Off-line host setup, part 1: fine pencil assembly and regular partitioning
(numpy/scipy restatement of proj/src/fine_grid.cpp:58-112 and
proj/src/partition.cpp:236-279,349-663).

This is the reference's *off-line* stage (``north_star``: "stays the
reference's host setup"); it is restated here only because the reference
cannot be compiled (Eigen absent) and desk-scale parity tests need real ROMs.
It is not on the hot path and runs on the host.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .._ffi import ConfigError, NumericalError


@dataclass
class Pencil:
    """SparsePencil (fine_grid.hpp:31-41): A (CSC, symmetric nonpositive),
    B (diagonal), grid dims and per-row coordinates."""
    A: sp.csc_matrix
    B: np.ndarray
    ndim: int
    dims: list
    coords: np.ndarray  # [n, 3]

    @property
    def n(self) -> int:
        return self.A.shape[0]

    def node_of(self, c) -> int:  # fine_grid.cpp:29-36 (row-major over dims)
        i = 0
        for a in range(self.ndim):
            if c[a] < 1 or c[a] > self.dims[a] - 2:
                return -1
            i = i * (self.dims[a] - 2) + (int(c[a]) - 1)
        return i

    def row_of_coord(self, c) -> int:
        """Row of a coordinate through `coords` (works on corner-modified
        pencils too); -1 if absent."""
        c = np.asarray(list(c) + [0] * (3 - len(c)))[:3]
        hits = np.nonzero(np.all(self.coords == c, axis=1))[0]
        return int(hits[0]) if hits.size else -1


def assemble_nd(medium) -> Pencil:
    """fine_grid.cpp:58-112 (same coefficient arithmetic)."""
    dims = list(medium.dims)
    nd = len(dims)
    if nd < 1 or nd > 3:
        raise ConfigError("medium must have 1-3 axes")
    if medium.h <= 0.0:
        raise ConfigError("grid step h must be positive")
    if any(d < 3 for d in dims):
        raise ConfigError("every axis needs at least 3 nodes (no interior otherwise)")
    sig = np.asarray(medium.sigma, np.float64)
    rho = np.asarray(medium.rho, np.float64)
    if np.any(sig < 0.0):
        raise ConfigError("sigma must be nonnegative")
    if np.any(rho <= 0.0):
        raise ConfigError("rho must be strictly positive")
    inv_h2 = 1.0 / (medium.h * medium.h)
    idims = [d - 2 for d in dims]
    n = int(np.prod(idims))
    coords = np.zeros((n, 3), np.int64)
    grids = np.meshgrid(*[np.arange(1, d - 1) for d in dims], indexing="ij")
    for a in range(nd):
        coords[:, a] = grids[a].reshape(-1)
    gstr = [int(np.prod(dims[a + 1:])) for a in range(nd)]
    istr = [int(np.prod(idims[a + 1:])) for a in range(nd)]
    gid = sum(coords[:, a] * gstr[a] for a in range(nd))
    B = rho[gid].copy()
    rows, cols, vals = [], [], []
    diag = np.zeros(n)
    rowids = np.arange(n)
    for a in range(nd):
        for d in (-1, 1):
            nb = gid + d * gstr[a]
            edge = 0.5 * (sig[gid] + sig[nb])
            diag = diag - edge * inv_h2
            ok = (coords[:, a] + d >= 1) & (coords[:, a] + d <= dims[a] - 2)
            rows.append(rowids[ok])
            cols.append(rowids[ok] + d * istr[a])
            vals.append(edge[ok] * inv_h2)
    rows.append(rowids)
    cols.append(rowids)
    vals.append(diag)
    A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    A.sort_indices()
    return Pencil(A, B, nd, dims, coords)


@dataclass
class Interface:
    ci: int
    cj: int
    nodes: np.ndarray  # sorted global ids


@dataclass
class HangingNode:
    id: int
    parent: int
    ci: int
    cj: int


@dataclass
class Partition:
    """partition.hpp:30-42."""
    n_nodes: int
    cells: list
    interiors: list = field(default_factory=list)
    boundaries: list = field(default_factory=list)
    interfaces: list = field(default_factory=list)
    skeleton: np.ndarray = None
    corner_set: np.ndarray = None
    hanging: list = field(default_factory=list)

    def num_cells(self) -> int:
        return len(self.cells)

    def cell_interfaces(self, c: int) -> list:
        return [f for f, I in enumerate(self.interfaces) if I.ci == c or I.cj == c]


@dataclass
class Split:
    """SubdomainSplit (partition.hpp:14-17): local A (CSC) and B."""
    A: sp.csc_matrix
    B: np.ndarray


def build_partition(n_nodes: int, cells: list) -> Partition:  # partition.cpp:236-275
    owners = [[] for _ in range(n_nodes)]
    for c, nodes in enumerate(cells):
        for g in nodes:
            owners[g].append(c)
    part = Partition(n_nodes, [np.asarray(c, np.int64) for c in cells])
    part.interiors = [[] for _ in cells]
    part.boundaries = [[] for _ in cells]
    iface = {}
    skel, corner = [], []
    for g in range(n_nodes):
        own = owners[g]
        if len(own) <= 1:
            if len(own) == 1:
                part.interiors[own[0]].append(g)
            continue
        skel.append(g)
        for c in own:
            part.boundaries[c].append(g)
        for i in range(len(own)):
            for j in range(i + 1, len(own)):
                iface.setdefault((own[i], own[j]), []).append(g)
        if len(own) >= 3:
            corner.append(g)
    part.interiors = [np.asarray(x, np.int64) for x in part.interiors]
    part.boundaries = [np.asarray(x, np.int64) for x in part.boundaries]
    part.interfaces = [Interface(k[0], k[1], np.asarray(v, np.int64)) for k, v in sorted(iface.items())]
    part.skeleton = np.asarray(skel, np.int64)
    part.corner_set = np.asarray(corner, np.int64)
    return part


def regular_partition(pencil: Pencil, cells_per_axis):  # partition.cpp:349-461
    nd = pencil.ndim
    cpa = list(cells_per_axis)
    if len(cpa) != nd:
        raise ConfigError("cells_per_axis must match the grid dimension")
    ln = [1, 1, 1]
    for a in range(nd):
        c = cpa[a]
        if c < 1:
            raise ConfigError("cells per axis must be >= 1")
        if (pencil.dims[a] - 1) % c != 0:
            raise ConfigError(f"cells per axis must divide the interval count of axis {a}")
        ln[a] = (pencil.dims[a] - 1) // c
        if c > 1 and ln[a] < 2:
            raise ConfigError(f"coarse cells thinner than two fine intervals on axis {a}")
    n = pencil.n

    def cell_id(cc):
        i = 0
        for a in range(nd):
            i = i * cpa[a] + cc[a]
        return i

    owners = []
    for g in range(n):
        axis_cells = []
        for a in range(nd):
            x = int(pencil.coords[g, a])
            k = x // ln[a]
            if x % ln[a] == 0:
                ac = []
                if k - 1 >= 0:
                    ac.append(k - 1)
                if k <= cpa[a] - 1:
                    ac.append(k)
                axis_cells.append(ac)
            else:
                axis_cells.append([min(k, cpa[a] - 1)])
        owners.append(sorted(cell_id(cc) for cc in itertools.product(*axis_cells)))
    n_cells = int(np.prod(cpa))
    cells = [[] for _ in range(n_cells)]
    for g in range(n):
        for c in owners[g]:
            cells[c].append(g)
    A = pencil.A.tocsc()
    A.sort_indices()
    # column k's entries straight from the CSC arrays (scipy's getcol is
    # ~100x slower and dominated the 129^3 partition)
    indptr, indices, data = A.indptr, A.indices.tolist(), A.data.tolist()

    def column(k):
        lo, hi = indptr[k], indptr[k + 1]
        return indices[lo:hi], data[lo:hi]

    splits = []
    for c in range(n_cells):
        nodes = cells[c]
        loc = {g: i for i, g in enumerate(nodes)}
        rr, cc_, vv = [], [], []
        s_local = np.zeros(len(nodes))
        Bc = np.zeros(len(nodes))
        for i, k in enumerate(nodes):
            Bc[i] = pencil.B[k] / len(owners[k])
            for l, v in zip(*column(k)):
                if l == k or l not in loc:
                    continue
                shared = len(set(owners[k]) & set(owners[l]))
                w = v / shared
                rr.append(i)
                cc_.append(loc[l])
                vv.append(w)
                s_local[i] += abs(w)
        for i, k in enumerate(nodes):
            ci_, cv_ = column(k)
            akk = next((v for l, v in zip(ci_, cv_) if l == k), 0.0)
            if len(owners[k]) == 1:
                rr.append(i)
                cc_.append(i)
                vv.append(akk)
            else:
                total = float(sum(abs(v) for l, v in zip(ci_, cv_) if l != k))
                share = s_local[i] / total if total > 0.0 else 1.0 / len(owners[k])
                rr.append(i)
                cc_.append(i)
                vv.append(akk * share)
        As = sp.csc_matrix((vv, (rr, cc_)), shape=(len(nodes), len(nodes)))
        splits.append(Split(As, Bc))
    return build_partition(n, cells), splits


def remove_corner_set(pencil: Pencil, part: Partition, splits):  # partition.cpp:463-663
    if part.corner_set.size == 0:
        return pencil, part, splits
    n = pencil.n
    is_corner = np.zeros(n, bool)
    is_corner[part.corner_set] = True
    nf = len(part.interfaces)
    survives = np.zeros(nf, bool)
    ifaces_of = [[] for _ in range(n)]
    for f, I in enumerate(part.interfaces):
        for g in I.nodes:
            ifaces_of[g].append(f)
            if not is_corner[g]:
                survives[f] = True
    compact = -np.ones(n, np.int64)
    next_id = 0
    for g in range(n):
        if not is_corner[g]:
            compact[g] = next_id
            next_id += 1
    copy_id = {}
    hanging = []
    for k in part.corner_set:
        any_ = False
        for f in ifaces_of[k]:
            if not survives[f]:
                continue
            copy_id[(int(k), f)] = next_id
            next_id += 1
            hanging.append(HangingNode(copy_id[(int(k), f)], int(k), part.interfaces[f].ci, part.interfaces[f].cj))
            any_ = True
        if not any_:
            raise NumericalError(f"corner node {k} has no surviving interface")

    def touches(f, cell):
        return part.interfaces[f].ci == cell or part.interfaces[f].cj == cell

    iface_sets = [set(I.nodes.tolist()) for I in part.interfaces]
    new_cells, new_splits = [], []
    for c in range(part.num_cells()):
        gnodes = part.cells[c]
        nc = len(gnodes)
        new_g = [int(compact[g]) for g in gnodes if not is_corner[g]]
        cell_copies = {}
        for g in gnodes:
            if not is_corner[g]:
                continue
            lst = [f for f in ifaces_of[g] if survives[f] and touches(f, c)]
            if not lst:
                raise NumericalError(f"corner node {g} has no surviving interface in cell {c}")
            cell_copies[int(g)] = lst
            new_g.extend(copy_id[(int(g), f)] for f in lst)
        new_g = sorted(new_g)
        new_cells.append(new_g)
        new_loc = {g: i for i, g in enumerate(new_g)}
        entries = {}

        def add_sym(a, b, v):
            entries[(a, b)] = entries.get((a, b), 0.0) + v
            entries[(b, a)] = entries.get((b, a), 0.0) + v

        old = splits[c].A.tocsc()
        old.sort_indices()
        o_ptr, o_idx, o_val = old.indptr, old.indices.tolist(), old.data.tolist()
        old_diag = np.zeros(nc)
        old_off = np.zeros(nc)
        for li in range(nc):
            gk = int(gnodes[li])
            for lj, v in zip(o_idx[o_ptr[li]:o_ptr[li + 1]], o_val[o_ptr[li]:o_ptr[li + 1]]):
                gl = int(gnodes[lj])
                if lj == li:
                    old_diag[li] = v
                    continue
                old_off[li] += abs(v)
                if gl < gk:
                    continue
                if not is_corner[gk] and not is_corner[gl]:
                    add_sym(new_loc[int(compact[gk])], new_loc[int(compact[gl])], v)
                elif is_corner[gk] != is_corner[gl]:
                    corner = gk if is_corner[gk] else gl
                    other = gl if is_corner[gk] else gk
                    copies = cell_copies[corner]
                    owner = next((f for f in copies if other in iface_sets[f]), -1)
                    if owner >= 0:
                        add_sym(new_loc[copy_id[(corner, owner)]], new_loc[int(compact[other])], v)
                    else:
                        share = v / len(copies)
                        for f in copies:
                            add_sym(new_loc[copy_id[(corner, f)]], new_loc[int(compact[other])], share)
                else:
                    placed = False
                    for f in cell_copies[gk]:
                        if gl not in iface_sets[f]:
                            continue
                        add_sym(new_loc[copy_id[(gk, f)]], new_loc[copy_id[(gl, f)]], v)
                        placed = True
                    if not placed:
                        raise NumericalError(f"adjacent corner nodes {gk},{gl} share no surviving interface")
        off_sum = np.zeros(len(new_g))
        for (r, _), v in entries.items():
            off_sum[r] += abs(v)
        rr = [k[0] for k in entries]
        cc_ = [k[1] for k in entries]
        vv = list(entries.values())
        Bn = np.zeros(len(new_g))
        for li in range(nc):
            gk = int(gnodes[li])
            if not is_corner[gk]:
                i = new_loc[int(compact[gk])]
                rr.append(i)
                cc_.append(i)
                vv.append(old_diag[li])
                Bn[i] = splits[c].B[li]
            else:
                copies = cell_copies[gk]
                deficit = old_diag[li] + old_off[li]
                for f in copies:
                    i = new_loc[copy_id[(gk, f)]]
                    rr.append(i)
                    cc_.append(i)
                    vv.append(-off_sum[i] + deficit / len(copies))
                    Bn[i] = splits[c].B[li]
        As = sp.csc_matrix((vv, (rr, cc_)), shape=(len(new_g), len(new_g)))
        new_splits.append(Split(As, Bn))
    npart = build_partition(next_id, new_cells)
    npart.hanging = hanging
    if npart.corner_set.size:
        raise NumericalError("corner removal left a nonempty corner set")
    coords = np.zeros((next_id, 3), np.int64)
    for g in range(n):
        if compact[g] >= 0:
            coords[compact[g]] = pencil.coords[g]
    for hn in hanging:
        coords[hn.id] = pencil.coords[hn.parent]
    rr, cc_, vv = [], [], []
    gB = np.zeros(next_id)
    for c, nodes in enumerate(new_cells):
        nodes = np.asarray(nodes)
        gB[nodes] += new_splits[c].B
        coo = new_splits[c].A.tocoo()
        rr.append(nodes[coo.row])
        cc_.append(nodes[coo.col])
        vv.append(coo.data)
    A = sp.csc_matrix((np.concatenate(vv), (np.concatenate(rr), np.concatenate(cc_))), shape=(next_id, next_id))
    A.sum_duplicates()
    A.sort_indices()
    return Pencil(A, gB, pencil.ndim, pencil.dims, coords), npart, new_splits
