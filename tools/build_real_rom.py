"""Build a REAL (off-line stage, not synthetic) 3-D ROM at BASELINE config-2
shape and write it in the reference's archive format (the input the on-line
B200 stepper loads with msw_create_from_archive).

Config 2 (BASELINE.json): 129^3 fine nodes, 8^3 coarse cells of 16^3, a
layered medium of 8 horizontal (axis-0) layers with seeded sigma ~ U[1,4],
rho ~ U[1,2] per layer; 16 point sources and 128 point receivers.  The
BASELINE's z = 4 plane is not on the skeleton, which the reference rejects
(romgen.cpp:463-475), so sources and receivers sit on the skeleton plane
z = 16, at face-interior nodes.  omega_max follows
"10 fine nodes per minimum wavelength": f_max = c_min / 10h.
M is pinned to <= 6 by max_basis_per_interface.  The collar Gramians exceed
the reference's 5000-node dense gate, so they use the in-band partial
eigensolver (RomOptions.gramian_solver = "auto").

Off-line host setup (numpy/scipy restatement of the reference's
partition.cpp / romgen.cpp), run once; writes <out>/manifest.json,
<out>/cell_*.bin and <out>/io.npz (projected sources / receivers and the
fine-grid rows of the same points).

  python tools/build_real_rom.py [--out data/rom_c2] [--workers N] [--cells 8 --cell-len 16]
"""
import argparse
import json
import math
import os
import sys
import time

# one BLAS / LAPACK thread per worker process: the per-interface and per-cell
# pools already use every core (oversubscription made the build ~20x slower)
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1604_06750_b200.archive import project_receivers, project_sources, write_rom_archive  # noqa: E402
from paper_1604_06750_b200.fine import node_of  # noqa: E402
from paper_1604_06750_b200.synthetic import layered_medium, lognormal_medium, skeleton_points  # noqa: E402
from paper_1604_06750_b200.offline import (RomOptions, assemble_nd, build_all_roms, build_boundary_basis,  # noqa: E402
                                           regular_partition, remove_corner_set)


def plane_points(dims, cell_len, plane, count, seed):
    rng = np.random.default_rng(seed)
    pts = set()
    while len(pts) < count:
        c = [plane]
        for a in (1, 2):
            while True:
                x = int(rng.integers(1, dims[a] - 1))
                if x % cell_len:
                    break
            c.append(x)
        pts.add(tuple(c))
    return sorted(pts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "data", "rom_c2"))
    ap.add_argument("--cells", type=int, default=8)
    ap.add_argument("--cell-len", type=int, default=16)
    ap.add_argument("--sources", type=int, default=16)
    ap.add_argument("--receivers", type=int, default=128)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--max-basis", type=int, default=6)
    ap.add_argument("--nodes-per-wavelength", type=float, default=10.0)
    ap.add_argument("--medium", choices=["layered", "lognormal"], default="layered",
                    help="layered: BASELINE config 2; lognormal: configs 3/5 (sources on any skeleton plane)")
    ap.add_argument("--c-ref", choices=["min", "p5"], default="min",
                    help="velocity for the nodes-per-wavelength rule: the minimum (BASELINE wording) or the 5th "
                         "percentile (a random lognormal field's extreme minimum leaves whole collars without "
                         "in-band modes, i.e. cells with an empty reduced boundary)")
    ap.add_argument("--partition-cache", default=None,
                    help="pickle file for the partition stage (reused when present)")
    args = ap.parse_args()
    t0 = time.time()
    n = args.cells * args.cell_len + 1
    dims = [n, n, n]
    if args.medium == "layered":
        med, sig_l, rho_l = layered_medium(dims)
        c_min = math.sqrt(sig_l.min() / rho_l.max())
    else:
        med = lognormal_medium(dims, seed=77)
        sig_l, rho_l = np.array([med.sigma.min()]), np.array([med.rho.max()])
        c_min = math.sqrt(float(med.sigma.min()) / float(med.rho.max()))
    if args.c_ref == "p5":
        c_min = float(np.quantile(np.sqrt(med.sigma / med.rho), 0.05))
    omega_max = 2.0 * math.pi * c_min / (args.nodes_per_wavelength * med.h)
    opt = RomOptions(m=4, omega_max=omega_max, epsilon_rel=1e-6, max_basis_per_interface=args.max_basis,
                     gramian_solver="auto", workers=args.workers)
    import pickle
    if args.partition_cache and os.path.exists(args.partition_cache):
        with open(args.partition_cache, "rb") as fh:
            pencil, part, splits = pickle.load(fh)
    else:
        orig = assemble_nd(med)
        part, splits = regular_partition(orig, [args.cells] * 3)
        pencil, part, splits = remove_corner_set(orig, part, splits)
        del orig
        if args.partition_cache:
            with open(args.partition_cache, "wb") as fh:
                pickle.dump((pencil, part, splits), fh, protocol=pickle.HIGHEST_PROTOCOL)
    t1 = time.time()
    if args.medium == "layered":
        plane = args.cell_len  # first interior skeleton plane
        pts = plane_points(dims, args.cell_len, plane, args.sources + args.receivers, seed=5)
    else:
        pts = [tuple(int(x) for x in p_) for p_ in
               skeleton_points(dims, args.cell_len, args.sources + args.receivers, seed=5)]
    rng = np.random.default_rng(9)
    order = rng.permutation(len(pts))
    src_pts = [pts[i] for i in order[:args.sources]]
    rcv_pts = [pts[i] for i in order[args.sources:]]
    rows_mod = lambda p: pencil.row_of_coord(p)
    vec = lambda r: (np.array([r], np.int64), np.array([1.0]))
    g0 = np.zeros(pencil.n)
    q0 = np.zeros(pencil.n)
    g0[rows_mod(src_pts[0])] = 1.0
    q0[rows_mod(rcv_pts[0])] = 1.0
    basis = build_boundary_basis(pencil, part, opt)
    t2 = time.time()
    empty = [f for f, S_f in enumerate(basis.S) if S_f.shape[1] == 0]
    if empty:  # the reference would throw in build_rom (romgen.cpp): stop before the ROM stage
        raise SystemExit(f"{len(empty)} interfaces kept no basis vector (omega_max {omega_max:.4g} too low "
                         f"for their collars); raise omega_max (--nodes-per-wavelength / --c-ref p5)")
    roms = build_all_roms(part, splits, basis, g0, q0, opt)
    t3 = time.time()
    write_rom_archive(args.out, roms, basis, opt)
    G = project_sources(part, basis, [vec(rows_mod(p)) for p in src_pts])
    rc = project_receivers(part, basis, [vec(rows_mod(p)) for p in rcv_pts])
    np.savez(os.path.join(args.out, "io.npz"), g=G, rcv_ptr=rc.rcv_ptr, rcv_iface=rc.term_iface, rcv_q=rc.term_q,
             fine_src_rows=np.array([node_of(dims, p) for p in src_pts], np.int64),
             fine_rcv_rows=np.array([node_of(dims, p) for p in rcv_pts], np.int64),
             src_pts=np.array(src_pts), rcv_pts=np.array(rcv_pts), dims=np.array(dims),
             sigma_layers=sig_l, rho_layers=rho_l, omega_max=omega_max)
    M = [s.shape[1] for s in basis.S]
    info = {"dims": dims, "cells": args.cells, "cell_len": args.cell_len, "interfaces": len(M),
            "medium": args.medium, "c_ref": args.c_ref, "c_used": c_min,
            "M_min": int(min(M)), "M_max": int(max(M)), "ktilde_max": int(max(r.ktilde for r in roms)),
            "omega_max": omega_max, "partition_s": t1 - t0, "basis_s": t2 - t1, "roms_s": t3 - t2,
            "total_s": time.time() - t0, "workers": args.workers}
    with open(os.path.join(args.out, "build_info.json"), "w") as f:
        json.dump(info, f, indent=1)
    print(json.dumps(info))


if __name__ == "__main__":
    main()
