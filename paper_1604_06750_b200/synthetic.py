"""Seeded, shape-faithful synthetic ROM systems for the BASELINE.json configs.

The reference's off-line stage cannot produce ROMs at configs 3/5 (the
two-cell-collar Gramian is gated at 5000 nodes, romgen.cpp:15,91-92, and
Eigen is absent here; SURVEY.md §7 "Hard parts").  The on-line kernels'
cost depends only on the shapes, so the throughput configs use systems with
exactly the reference's structure:

* a regular cells_per_axis^3 partition after corner removal: interfaces are
  the face-adjacent cell pairs (ci < cj) in lexicographic (ci, cj) order
  (build_partition, partition.cpp:236-275); every cell lists its interfaces
  ascending with M-sized blocks (romgen.cpp:404-412);
* m = 4 S-fraction layers (RomOptions default, romgen.hpp:121);
* SPD ladders L^k, Lhat^k (exactly symmetric, as romgen.cpp:279,284
  symmetrises them) with spectra in a fixed band;
* point sources / receivers on face-interior skeleton nodes: g~_f = S_f^T e_k
  is one row of an orthonormal K_f x M basis, emulated by a random row of
  norm ~ sqrt(M/K_f).

Both the GPU path and the oracle consume the same arrays, so parity does not
depend on how the ROM was produced (SURVEY.md §7 "Minimum slice").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rom import FlatSystem, Receivers

# BASELINE.json configs as the reference needs them.
CONFIGS = {
    "c1": dict(cells=(8, 8, 8), cell_len=8, M=1, m=4, S=1, R=64, steps=2000, fine_dims=(65, 65, 65)),
    "c2": dict(cells=(8, 8, 8), cell_len=16, M=6, m=4, S=16, R=128, steps=3000, fine_dims=(129, 129, 129)),
    "c3": dict(cells=(16, 16, 16), cell_len=16, M=6, m=4, S=64, R=256, steps=4000, fine_dims=(257, 257, 257)),
    "c5": dict(cells=(16, 16, 16), cell_len=24, M=17, m=4, S=128, R=512, steps=1000, fine_dims=(385, 385, 385)),
}


def regular_topology(cells_per_axis):
    """Face-adjacent interfaces of a regular cell grid (row-major cell ids,
    axis 0 slowest).  Returns (pairs [nf,2] sorted by (ci,cj), per-cell
    ascending interface lists)."""
    cpa = list(cells_per_axis)
    nd = len(cpa)
    nc = int(np.prod(cpa))
    strides = [int(np.prod(cpa[a + 1:])) for a in range(nd)]
    coords = np.stack(np.unravel_index(np.arange(nc), cpa), axis=1)
    pairs = []
    for a in range(nd):
        ok = coords[:, a] < cpa[a] - 1
        ci = np.nonzero(ok)[0]
        pairs.append(np.stack([ci, ci + strides[a]], axis=1))
    pairs = np.concatenate(pairs)
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    pairs = pairs[order]
    cell_ifaces = [[] for _ in range(nc)]
    for f, (i, j) in enumerate(pairs):
        cell_ifaces[i].append(f)
        cell_ifaces[j].append(f)
    for lst in cell_ifaces:
        lst.sort()
    return pairs, cell_ifaces


def _spd_batch(rng, count, n, lo, hi):
    """count random SPD n x n matrices with spectra in ~[lo, hi], exactly
    symmetric (0.5 (A + A^T))."""
    G = rng.standard_normal((count, n, n))
    W = G @ np.swapaxes(G, 1, 2) / (4.0 * n)  # spectrum ~ [0, 1]
    A = lo * np.eye(n) + (hi - lo) * W
    return 0.5 * (A + np.swapaxes(A, 1, 2))


@dataclass
class SyntheticCase:
    flat: FlatSystem
    g: np.ndarray           # [total_io, S]
    receivers: Receivers
    src_iface: np.ndarray   # interface of each source
    rcv_iface: np.ndarray
    dt: float
    lam_bound: float
    config: dict


def synthetic_system(cells_per_axis, M: int, m: int = 4, S: int = 1, R: int = 1, seed: int = 0,
                     K_face: int = 289, band=(0.5, 2.0), hat_band=(0.5, 2.0),
                     safety: float = 0.9) -> SyntheticCase:
    rng = np.random.default_rng(seed)
    pairs, cell_ifaces = regular_topology(cells_per_axis)
    nc = len(cell_ifaces)
    nf = pairs.shape[0]
    cell_kt = np.array([len(l) * M for l in cell_ifaces], np.int32)
    cell_m = np.full(nc, m, np.int32)
    ptr_ = np.concatenate([[0], np.cumsum([len(l) for l in cell_ifaces])]).astype(np.int32)
    ids = np.concatenate([np.asarray(l, np.int32) for l in cell_ifaces])
    offs = np.concatenate([np.arange(len(l), dtype=np.int32) * M for l in cell_ifaces])
    sizes = (2 * m * cell_kt.astype(np.int64) ** 2)
    lad_off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    ladders = np.empty(int(sizes.sum()))
    # ladders, batched per ktilde
    inf_L = np.zeros((nc, m))
    inf_H = np.zeros((nc, m))
    rowinf_L1 = [None] * nc
    for kt in np.unique(cell_kt):
        cs = np.nonzero(cell_kt == kt)[0]
        L = _spd_batch(rng, len(cs) * m, int(kt), *band).reshape(len(cs), m, kt, kt)
        H = _spd_batch(rng, len(cs) * m, int(kt), *hat_band).reshape(len(cs), m, kt, kt)
        both = np.concatenate([L, H], axis=1)  # [cells, 2m, kt, kt]
        colmajor = np.swapaxes(both, 2, 3).reshape(len(cs), -1)
        for t, c in enumerate(cs):
            o = lad_off[c]
            ladders[o:o + colmajor.shape[1]] = colmajor[t]
        inf_L[cs] = np.abs(L).sum(axis=3).max(axis=2)
        inf_H[cs] = np.abs(H).sum(axis=3).max(axis=2)
        rs = np.abs(L[:, 0]).sum(axis=2)  # row abs sums of L^1, [cells, kt]
        for t, c in enumerate(cs):
            rowinf_L1[c] = rs[t]
    li = np.zeros(nf, np.int32)
    lj = np.zeros(nf, np.int32)
    for f, (i, j) in enumerate(pairs):
        li[f] = cell_ifaces[i].index(f)
        lj[f] = cell_ifaces[j].index(f)
    flat = FlatSystem(cell_m, cell_kt, ptr_, ids, offs, lad_off, ladders, pairs[:, 0], pairs[:, 1],
                      li, lj, np.full(nf, M, np.int32))
    # stability bound: lambda_max <= ||K||_inf (any induced norm)
    lam_int = 0.0
    if m > 1:
        for k in range(1, m):
            lam_int = max(lam_int, float(np.max(inf_H[:, k] * 2.0 * (inf_L[:, k] + inf_L[:, k - 1]))))
    # interfaces: mass = [inv(H1_i[f,f]) + inv(H1_j[f,f])]^-1 (host numpy, bound only)
    lam_if = 0.0
    H1_blocks_i = np.empty((nf, M, M))
    H1_blocks_j = np.empty((nf, M, M))
    for f, (i, j) in enumerate(pairs):
        for blocks, c, l in ((H1_blocks_i, i, li[f]), (H1_blocks_j, j, lj[f])):
            kt = int(cell_kt[c])
            o = int(lad_off[c]) + m * kt * kt
            H1 = ladders[o:o + kt * kt].reshape(kt, kt).T
            b = l * M
            blocks[f] = H1[b:b + M, b:b + M]
    mass = np.linalg.inv(np.linalg.inv(H1_blocks_i) + np.linalg.inv(H1_blocks_j))
    mass_inf = np.abs(mass).sum(axis=2).max(axis=1)
    for f, (i, j) in enumerate(pairs):
        ri = rowinf_L1[i][li[f] * M:(li[f] + 1) * M].max()
        rj = rowinf_L1[j][lj[f] * M:(lj[f] + 1) * M].max()
        lam_if = max(lam_if, float(mass_inf[f] * 2.0 * (ri + rj)))
    lam = max(lam_int, lam_if)
    dt = safety * 2.0 / np.sqrt(lam)
    # sources / receivers: one face-interior node each
    total_io = nf * M
    src_iface = rng.integers(0, nf, size=S)
    g = np.zeros((total_io, S))
    for s in range(S):
        f = src_iface[s]
        g[f * M:(f + 1) * M, s] = rng.standard_normal(M) / np.sqrt(K_face)
    rcv_iface = np.sort(rng.integers(0, nf, size=R)) if R > 0 else np.zeros(0, np.int64)
    terms = [[(int(f), rng.standard_normal(M) / np.sqrt(K_face))] for f in rcv_iface]
    return SyntheticCase(flat, g, Receivers.from_terms(terms), src_iface, rcv_iface, float(dt),
                         float(lam), dict(cells=tuple(cells_per_axis), M=M, m=m, S=S, R=R, seed=seed))


def config_case(name: str, S: int | None = None, seed: int = 1234) -> SyntheticCase:
    cfg = CONFIGS[name]
    return synthetic_system(cfg["cells"], cfg["M"], cfg["m"], S or cfg["S"], cfg["R"], seed=seed,
                            K_face=(cfg["cell_len"] - 1) ** 2)


def lognormal_medium(dims, seed: int = 0, mean: float = 2.0, log_std: float = 0.3,
                     corr_len: float = 3.0, n_spheres: int = 200, r_range=(2.0, 6.0),
                     contrast: float = 3.0, rho_range=(1.0, 1.5), h: float = 1.0):
    """BASELINE config 3/5 medium (seeded synthetic stand-in): lognormal sigma
    with mean `mean`, log-std `log_std`, Gaussian-filtered to correlation
    length `corr_len` nodes, plus `n_spheres` spherical inclusions of radius
    in r_range with sigma x contrast; rho ~ U[rho_range] per node."""
    from scipy.ndimage import gaussian_filter

    from .fine import GridMedium

    rng = np.random.default_rng(seed)
    dims = list(dims)
    z = rng.standard_normal(dims)
    z = gaussian_filter(z, sigma=corr_len, mode="wrap")
    z /= max(z.std(), 1e-300)
    mu = np.log(mean) - 0.5 * log_std ** 2
    sigma = np.exp(mu + log_std * z)
    for _ in range(n_spheres):
        c = [rng.uniform(0, d - 1) for d in dims]
        r = rng.uniform(*r_range)
        lo = [max(0, int(np.floor(ci - r))) for ci in c]
        hi = [min(d, int(np.ceil(ci + r)) + 1) for ci, d in zip(c, dims)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        grids = np.meshgrid(*[np.arange(a, b) for a, b in zip(lo, hi)], indexing="ij")
        d2 = sum((g - ci) ** 2 for g, ci in zip(grids, c))
        block = sigma[sl]
        block[d2 <= r * r] *= contrast
    rho = rng.uniform(rho_range[0], rho_range[1], size=dims)
    return GridMedium(dims, h, np.ascontiguousarray(sigma.reshape(-1)), np.ascontiguousarray(rho.reshape(-1)))


def layered_medium(dims, n_layers: int = 8, seed: int = 2, h: float = 1.0):
    """BASELINE config 2 medium (seeded synthetic stand-in): n_layers
    horizontal layers along axis 0 with sigma ~ U[1, 4] and rho ~ U[1, 2] per
    layer.  Returns (GridMedium, sigma per layer, rho per layer)."""
    from .fine import GridMedium

    rng = np.random.default_rng(seed)
    sig_l = rng.uniform(1.0, 4.0, n_layers)
    rho_l = rng.uniform(1.0, 2.0, n_layers)
    dims = list(dims)
    layer = np.minimum(n_layers - 1, np.arange(dims[0]) * n_layers // dims[0])
    shape = (dims[0],) + (1,) * (len(dims) - 1)
    sig = np.broadcast_to(sig_l[layer].reshape(shape), dims).reshape(-1).copy()
    rho = np.broadcast_to(rho_l[layer].reshape(shape), dims).reshape(-1).copy()
    return GridMedium(dims, h, sig, rho), sig_l, rho_l


def skeleton_points(dims, cell_len: int, count: int, seed: int = 0):
    """`count` distinct face-interior skeleton nodes of a regular partition
    with cells of `cell_len` intervals (a coordinate on a skeleton plane,
    the other two strictly inside a cell): the only legal source/receiver
    positions after corner removal (romgen.cpp:463-475)."""
    rng = np.random.default_rng(seed)
    nd = len(dims)
    pts = set()
    while len(pts) < count:
        a = int(rng.integers(0, nd))
        c = []
        for b in range(nd):
            ncell = (dims[b] - 1) // cell_len
            if b == a:
                c.append(int(rng.integers(1, ncell)) * cell_len)  # interior skeleton plane
            else:
                k = int(rng.integers(0, ncell))
                c.append(k * cell_len + int(rng.integers(1, cell_len)))
        pts.add(tuple(c) + (0,) * (3 - nd))
    return sorted(pts)
