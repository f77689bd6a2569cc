"""Off-line host setup, part 2: per-cell ROM construction (numpy/scipy
restatement of proj/src/romgen.cpp) and assemble_system (msolver.cpp:31-106).

Off-line stage only (see partition.py).  Dense linear algebra at desk scale;
numerical conventions follow the reference: thin QR with a nonnegative R
diagonal (romgen.cpp:20-38), eigenvectors signed so the largest-magnitude
entry is positive (romgen.cpp:146-149), every ladder symmetrised
(romgen.cpp:279,284).  Results are property-matched to the reference (Eigen's
solvers are not bit-reproducible here), which is all the on-line parity
needs: the GPU stepper and the oracle consume the same ROM arrays.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .._ffi import ConfigError, NumericalError
from ..rom import CornerCopy, CornerGroup, CoupledInterface, FlatSystem, MultiscaleSystem, SubdomainROM

DENSE_ORACLE_LIMIT = 5000  # romgen.cpp:15


@dataclass
class RomOptions:  # romgen.hpp:120-127
    m: int = 4
    omega_max: float = 2.0 * 3.14159265358979323846
    epsilon_rel: float = 1e-6
    max_basis_per_interface: int = 0
    shift: float = 0.0
    full_collar: bool = False
    # B200 addition (off-line only): "dense" keeps the reference's gated full
    # eigensolve; "partial" lifts the gate (in-band shift-invert Lanczos);
    # "auto" = dense up to DENSE_ORACLE_LIMIT collar nodes, partial above
    gramian_solver: str = "dense"
    workers: int = 1  # process pool for the per-interface / per-cell loops


@dataclass
class BoundaryBasis:  # romgen.hpp:13-19
    omega_max: float = 0.0
    epsilon: float = 0.0
    S: list = field(default_factory=list)
    kept_eigs: list = field(default_factory=list)
    tail: list = field(default_factory=list)


def sym(m):
    return 0.5 * (m + m.T)


def thin_qr(block, who):  # romgen.cpp:20-38
    Q, R = np.linalg.qr(block, mode="reduced")
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    Q = Q * d
    R = R * d[:, None]
    scale = np.max(np.abs(R)) if R.size else 0.0
    for i in range(R.shape[1]):
        if not (R[i, i] > scale * 1e-13):
            raise NumericalError(f"{who}: block rank deficient (deflation needed), pivot {i}")
    return Q, R


def local_indices(nodes, subset):  # romgen.cpp:50-60
    nodes = np.asarray(nodes)
    pos = np.searchsorted(nodes, subset)
    if np.any(pos >= nodes.size) or np.any(nodes[np.minimum(pos, nodes.size - 1)] != subset):
        raise ConfigError("subset node not in the cell")
    return pos


def boundary_gramian(A, B, iface_nodes, omega_max, collar, solver="dense"):  # romgen.cpp:88-124
    """G = W W^T, W = the B^-1/2-scaled collar eigenvectors of (-A, B) with
    eigenvalue <= omega_max^2, restricted to the interface rows.

    solver="dense" is the reference's route: a full eigendecomposition,
    gated at DENSE_ORACLE_LIMIT collar nodes (romgen.cpp:15,91-92).
    solver="partial" lifts the gate: only the in-band eigenpairs are computed,
    by shift-invert Lanczos (scipy eigsh, sigma = 0) on the sparse collar
    operator, growing the number requested until one falls outside the band.
    G depends only on the in-band invariant subspace, so both routes agree to
    the eigensolvers' accuracy (tests/test_offline.py)."""
    nc = len(collar)
    pos = local_indices(collar, iface_nodes)
    dinv = 1.0 / np.sqrt(B[collar])
    w2 = omega_max * omega_max
    if solver == "dense":
        if nc > DENSE_ORACLE_LIMIT:
            raise ConfigError("boundary_gramian surrogate too large for the dense eigensolve")
        C = -A[np.ix_(collar, collar)].toarray()
        C = sym(dinv[:, None] * C * dinv[None, :])
        lam, V = np.linalg.eigh(C)
        keep = lam <= w2
        W = dinv[pos][:, None] * V[np.ix_(pos, np.nonzero(keep)[0])]
        return W @ W.T
    if solver != "partial":
        raise ConfigError(f"unknown Gramian solver {solver}")
    Cs = -A[collar][:, collar]
    Cs = sp.diags(dinv) @ Cs @ sp.diags(dinv)
    Cs = (0.5 * (Cs + Cs.T)).tocsc()
    # one sparse LU of the collar operator serves every restart
    lu = spla.splu(Cs)
    OPinv = spla.LinearOperator(Cs.shape, matvec=lu.solve, dtype=np.float64)
    k = min(16, nc - 2)
    while True:
        lam, V = spla.eigsh(Cs, k=k, sigma=0.0, which="LM", tol=0.0, OPinv=OPinv)
        if lam.max() > w2 or k >= nc - 2:
            break
        k = min(2 * k, nc - 2)
    keep = np.nonzero(lam <= w2)[0]
    W = dinv[pos][:, None] * V[np.ix_(pos, keep)]
    return W @ W.T


def truncate_basis(G, epsilon, max_cols=0):  # romgen.cpp:126-154
    lam, V = np.linalg.eigh(sym(G))
    K = G.shape[0]
    lam_max = max(0.0, lam.max()) if K else 0.0
    thr = epsilon * lam_max
    keep, tail = [], 0.0
    for l in range(K - 1, -1, -1):
        if lam[l] > thr and (max_cols == 0 or len(keep) < max_cols):
            keep.append(l)
        else:
            tail += max(0.0, lam[l])
    S = np.zeros((K, len(keep)))
    kept = np.zeros(len(keep))
    for j, l in enumerate(keep):
        col = V[:, l].copy()
        if col[np.argmax(np.abs(col))] < 0.0:
            col = -col
        S[:, j] = col
        kept[j] = lam[l]
    return S, kept, tail


def rational_krylov(split, PS, s, m):  # romgen.cpp:156-188
    if s >= 0.0:
        raise ConfigError("rational Krylov shift must be negative")
    n, kt = PS.shape
    if m * kt > n:
        raise NumericalError("rational Krylov space larger than the cell (deflation needed)")
    if np.max(np.abs(PS.T @ PS - np.eye(kt))) > 1e-10:
        raise ConfigError("boundary input block is not orthonormal")
    M = (-split.A - s * sp.diags(split.B)).tocsc()
    lu = spla.splu(M)
    V = np.zeros((n, m * kt))
    V[:, :kt] = PS
    for k in range(1, m):
        Z = lu.solve(np.ascontiguousarray(V[:, (k - 1) * kt:k * kt]))
        for _ in range(2):
            Vp = V[:, :k * kt]
            Z = Z - Vp @ (Vp.T @ Z)
        Q, _ = thin_qr(Z, "rational_krylov")
        V[:, k * kt:(k + 1) * kt] = Q
    return V


def project_pencil(split, V, PS):  # romgen.cpp:190-196
    Am = sym(V.T @ (split.A @ V))
    Bm = sym(V.T @ (split.B[:, None] * V))
    Sm = V.T @ PS
    return Am, Bm, Sm


def block_lanczos(Am, Bm, Sm, m, kt):  # romgen.cpp:198-255
    n = Am.shape[0]
    if n != m * kt:
        raise ConfigError("block_lanczos: projected pencil size does not match m * ktilde")
    try:
        L = np.linalg.cholesky(Bm)
    except np.linalg.LinAlgError:
        raise NumericalError("block_lanczos: Bm not SPD")
    half = sla.solve_triangular(L, Am, lower=True)
    Atil = sym(sla.solve_triangular(L, half.T, lower=True))
    Stil = sla.solve_triangular(L, Sm, lower=True)
    Q = np.zeros((n, n))
    alphas, betas = [None] * m, [None] * m
    Q1, beta1 = thin_qr(Stil, "block_lanczos")
    Q[:, :kt] = Q1
    betas[0] = beta1
    for k in range(m):
        Qk = Q[:, k * kt:(k + 1) * kt]
        Z = Atil @ Qk
        if k > 0:
            Z = Z - Q[:, (k - 1) * kt:k * kt] @ betas[k].T
        alphas[k] = sym(Qk.T @ Z)
        Z = Z - Qk @ alphas[k]
        for _ in range(2):
            Vp = Q[:, :(k + 1) * kt]
            Z = Z - Vp @ (Vp.T @ Z)
        if k + 1 < m:
            Qn, R = thin_qr(Z, "block_lanczos")
            Q[:, (k + 1) * kt:(k + 2) * kt] = Qn
            betas[k + 1] = R
    T = np.zeros((n, n))
    for k in range(m):
        T[k * kt:(k + 1) * kt, k * kt:(k + 1) * kt] = alphas[k]
        if k + 1 < m:
            T[(k + 1) * kt:(k + 2) * kt, k * kt:(k + 1) * kt] = betas[k + 1]
            T[k * kt:(k + 1) * kt, (k + 1) * kt:(k + 2) * kt] = betas[k + 1].T
    return T, beta1


def sfraction_coeffs(T, beta1, m, kt):  # romgen.cpp:257-290
    hat, main = [], []
    G = beta1.T.copy()
    Lprev = np.zeros((kt, kt))
    for k in range(m):
        if k > 0:
            Ginv = np.linalg.inv(G)
            beta_k = T[k * kt:(k + 1) * kt, (k - 1) * kt:k * kt]
            G = np.linalg.solve(Lprev, Ginv.T @ beta_k.T)
        h = sym(G @ G.T)
        if np.linalg.eigvalsh(h).min() <= 0.0:
            raise NumericalError(f"sfraction_coeffs (hat): ladder entry {k + 1} is not SPD")
        hat.append(h)
        Ginv = np.linalg.inv(G)
        Lk = sym(-(Ginv.T @ T[k * kt:(k + 1) * kt, k * kt:(k + 1) * kt] @ Ginv) - Lprev)
        if np.linalg.eigvalsh(Lk).min() <= 0.0:
            raise NumericalError(f"sfraction_coeffs: ladder entry {k + 1} is not SPD")
        main.append(Lk)
        Lprev = Lk
    return hat, main


def evaluate_sfraction(hat, main, w2):  # romgen.cpp:294-331
    m = len(main)
    kt = main[0].shape[0]
    n = m * kt
    M = np.zeros((n, n), dtype=complex)
    for k in range(m):
        hinv = np.linalg.inv(hat[k])
        d = w2 * hinv - main[k]
        if k > 0:
            d = d - main[k - 1]
        M[k * kt:(k + 1) * kt, k * kt:(k + 1) * kt] = d
        if k + 1 < m:
            M[k * kt:(k + 1) * kt, (k + 1) * kt:(k + 2) * kt] = main[k]
            M[(k + 1) * kt:(k + 2) * kt, k * kt:(k + 1) * kt] = main[k]
    rhs = np.zeros((n, kt), dtype=complex)
    rhs[:kt, :kt] = np.eye(kt)
    return np.linalg.solve(M, rhs)[:kt]


def resolvent_transfer(T, beta1, w2):  # romgen.cpp:347-357
    n, kt = T.shape[0], beta1.shape[0]
    rhs = np.zeros((n, kt), dtype=complex)
    rhs[:kt] = beta1
    sol = np.linalg.solve(T + w2 * np.eye(n), rhs)
    return beta1.T @ sol[:kt]


def build_boundary_basis(pencil, part, opt: RomOptions) -> BoundaryBasis:  # romgen.cpp:365-396
    if opt.omega_max <= 0.0:
        raise ConfigError("omega_max must be positive")
    bb = BoundaryBasis(opt.omega_max, opt.epsilon_rel)
    A = pencil.A.tocsr()
    jobs = []
    for I in part.interfaces:
        if opt.full_collar:
            collar = np.arange(pencil.n)
        else:
            collar = np.union1d(part.cells[I.ci], part.cells[I.cj])
        solver = opt.gramian_solver
        if solver == "auto":
            solver = "dense" if len(collar) <= DENSE_ORACLE_LIMIT else "partial"
        jobs.append((I.nodes, collar, solver))
    if opt.workers > 1 and len(jobs) > 1:
        from concurrent.futures import ProcessPoolExecutor
        global _POOL_STATE
        _POOL_STATE = (A, pencil.B, opt)
        import multiprocessing as mp
        with ProcessPoolExecutor(opt.workers, mp_context=mp.get_context("fork")) as ex:
            results = list(ex.map(_basis_job, jobs, chunksize=1))
        _POOL_STATE = None
    else:
        results = [_basis_one(A, pencil.B, opt, *j) for j in jobs]
    for S, kept, tail in results:
        bb.S.append(S)
        bb.kept_eigs.append(kept)
        bb.tail.append(tail)
    return bb


_POOL_STATE = None  # (A, B, opt) inherited by forked workers


def _basis_one(A, B, opt, nodes, collar, solver):
    import time
    t0 = time.perf_counter()
    G = boundary_gramian(A, B, nodes, opt.omega_max, collar, solver)
    out = truncate_basis(G, opt.epsilon_rel, opt.max_basis_per_interface)
    dt = time.perf_counter() - t0
    if dt > 20.0:
        import sys
        print(f"boundary_gramian: slow interface ({len(collar)} collar nodes, {dt:.1f} s)", file=sys.stderr, flush=True)
    return out


def _basis_job(job):
    A, B, opt = _POOL_STATE
    return _basis_one(A, B, opt, *job)


def build_rom(cell, part, splits, basis, g, q, opt: RomOptions) -> SubdomainROM:  # romgen.cpp:398-457
    rom = SubdomainROM(cell=cell, m=opt.m)
    rom.iface_ids = part.cell_interfaces(cell)
    if not rom.iface_ids:
        raise ConfigError(f"cell {cell} has no interfaces")
    offs = [0]
    for f in rom.iface_ids:
        offs.append(offs[-1] + basis.S[f].shape[1])
    rom.iface_offsets = offs
    rom.ktilde = offs[-1]
    if rom.ktilde == 0:
        raise ConfigError(f"cell {cell} has an empty reduced boundary (raise omega_max or epsilon)")
    nodes = part.cells[cell]
    split = splits[cell]
    PS = np.zeros((split.A.shape[0], rom.ktilde))
    for li, f in enumerate(rom.iface_ids):
        rows = local_indices(nodes, part.interfaces[f].nodes)
        S = basis.S[f]
        PS[rows, offs[li]:offs[li] + S.shape[1]] = S
    rom.shift = opt.shift if opt.shift != 0.0 else -(opt.omega_max / 4.0) ** 2
    if rom.shift >= 0.0:
        raise ConfigError("shift must be negative")
    rom.V = rational_krylov(split, PS, rom.shift, rom.m)
    rom.Am, rom.Bm, rom.Sm = project_pencil(split, rom.V, PS)
    rom.T, rom.beta1 = block_lanczos(rom.Am, rom.Bm, rom.Sm, rom.m, rom.ktilde)
    rom.ladder_hat, rom.ladder = sfraction_coeffs(rom.T, rom.beta1, rom.m, rom.ktilde)
    for f in rom.iface_ids:
        nd = part.interfaces[f].nodes
        rom.g_proj.append(basis.S[f].T @ g[nd])
        rom.q_proj.append(basis.S[f].T @ q[nd])
    return rom


def build_all_roms(part, splits, basis, g, q, opt: RomOptions):  # romgen.cpp:459-504
    on = np.zeros(part.n_nodes, bool)
    on[part.skeleton] = True
    for name, v in (("source", g), ("receiver", q)):
        bad = np.nonzero((np.asarray(v) != 0.0) & ~on)[0]
        if bad.size:
            raise ConfigError(f"{name} has support off the partition skeleton at nodes: "
                              + " ".join(str(int(b)) for b in bad))
    if opt.workers > 1 and part.num_cells() > 1:
        from concurrent.futures import ProcessPoolExecutor
        import multiprocessing as mp
        global _POOL_STATE
        _POOL_STATE = (part, splits, basis, g, q, opt)
        n = part.num_cells()
        with ProcessPoolExecutor(opt.workers, mp_context=mp.get_context("fork")) as ex:
            roms = list(ex.map(_rom_job, range(n), chunksize=1))
        _POOL_STATE = None
        return roms
    return [build_rom(c, part, splits, basis, g, q, opt) for c in range(part.num_cells())]


def _rom_job(c):
    part, splits, basis, g, q, opt = _POOL_STATE
    return build_rom(c, part, splits, basis, g, q, opt)


def assemble_system(part, basis, roms, B_diag) -> MultiscaleSystem:  # msolver.cpp:31-106
    sys = MultiscaleSystem(roms=roms)
    for f, pf in enumerate(part.interfaces):
        S = basis.S[f]
        M = S.shape[1]
        ri, rj = roms[pf.ci], roms[pf.cj]
        if f not in ri.iface_ids or f not in rj.iface_ids:
            raise ConfigError(f"cell is missing interface {f}")
        li, lj = ri.iface_ids.index(f), rj.iface_ids.index(f)
        if ri.block_size(li) != M or rj.block_size(lj) != M:
            raise ConfigError(f"mismatched interface bases between cells {pf.ci} and {pf.cj}")
        if np.any(ri.g_proj[li] != rj.g_proj[lj]) or np.any(ri.q_proj[li] != rj.q_proj[lj]):
            raise ConfigError(f"projected I/O disagrees between the two sides of interface {f}")
        oi, oj = ri.block_offset(li), rj.block_offset(lj)
        Mi = ri.ladder_hat[0][oi:oi + M, oi:oi + M]
        Mj = rj.ladder_hat[0][oj:oj + M, oj:oj + M]
        form = sym(np.linalg.inv(Mi) + np.linalg.inv(Mj))
        mass = sym(np.linalg.inv(form))
        sys.ifaces.append(CoupledInterface(part_iface=f, ci=pf.ci, cj=pf.cj, li=li, lj=lj, size=M, S=S,
                                           mass=mass, mass_form=form, g_proj=ri.g_proj[li].copy(),
                                           q_proj=ri.q_proj[li].copy()))
    groups = {}
    for hn in part.hanging:
        f = -1
        for i, I in enumerate(part.interfaces):
            if I.ci == hn.ci and I.cj == hn.cj and hn.id in set(I.nodes.tolist()):
                f = i
                break
        if f < 0:
            raise ConfigError("hanging node without a matching interface")
        row = int(np.searchsorted(part.interfaces[f].nodes, hn.id))
        groups.setdefault(hn.parent, CornerGroup(parent=hn.parent)).copies.append(
            CornerCopy(f, row, float(B_diag[hn.id])))
    sys.corners = [groups[k] for k in sorted(groups)]
    return sys


def corner_arrays(sys: MultiscaleSystem):
    """Flat corner description for msw_set_corners / oracle_set_corners."""
    gp, ci, cr, cm = [0], [], [], []
    for g in sys.corners:
        for c in g.copies:
            ci.append(c.iface)
            cr.append(c.row)
            cm.append(c.mass)
        gp.append(len(ci))
    K = [f.S.shape[0] for f in sys.ifaces]
    basis = np.concatenate([np.asarray(f.S, np.float64).T.reshape(-1) for f in sys.ifaces])
    return gp, ci, cr, cm, K, basis
