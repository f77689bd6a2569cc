"""Off-line host setup (the reference's partition + ROM build), restated in
numpy/scipy for desk-scale systems because the reference cannot be compiled
here (Eigen absent).  Not on the hot path; produces the real ROMs that the
parity tests feed to the B200 stepper and to the oracle alike."""
from dataclasses import dataclass

import numpy as np

from ..fine import make_uniform_medium
from ..rom import FlatSystem, system_receiver, system_sources
from .partition import (HangingNode, Interface, Partition, Pencil, Split, assemble_nd,  # noqa: F401
                        build_partition, regular_partition, remove_corner_set)
from .romgen import (BoundaryBasis, RomOptions, assemble_system, build_all_roms,  # noqa: F401
                     build_boundary_basis, build_rom, corner_arrays, evaluate_sfraction,
                     resolvent_transfer, sfraction_coeffs)


@dataclass
class BuiltSystem:
    """test_helpers.hpp:13-21."""
    pencil: Pencil            # corner-modified
    original_pencil: Pencil   # for fine references
    partition: Partition
    splits: list
    basis: BoundaryBasis
    system: object
    g: np.ndarray
    q: np.ndarray

    def flat(self) -> FlatSystem:
        return FlatSystem.from_system(self.system)

    def sources(self):
        return system_sources(self.system)

    def receiver(self):
        return system_receiver(self.system)


def build_regular(dims, h, cells_per_axis, opt: RomOptions, src, rcv, sigma=1.0, medium=None) -> BuiltSystem:
    """test_helpers.hpp:25-44: full off-line pipeline on a regular partition
    with corner removal; source/receiver point vectors on the modified
    pencil (looked up through coords)."""
    med = medium if medium is not None else make_uniform_medium(list(dims), h, sigma)
    orig = assemble_nd(med)
    part, splits = regular_partition(orig, cells_per_axis)
    pencil, part, splits = remove_corner_set(orig, part, splits)
    basis = build_boundary_basis(pencil, part, opt)
    g = np.zeros(pencil.n)
    q = np.zeros(pencil.n)
    gi = pencil.row_of_coord(src)
    qi = pencil.row_of_coord(rcv)
    if gi < 0 or qi < 0:
        from .._ffi import ConfigError
        raise ConfigError("source/receiver location has no node in the modified pencil")
    g[gi] = 1.0
    q[qi] = 1.0
    roms = build_all_roms(part, splits, basis, g, q, opt)
    system = assemble_system(part, basis, roms, pencil.B)
    return BuiltSystem(pencil, orig, part, splits, basis, system, g, q)
