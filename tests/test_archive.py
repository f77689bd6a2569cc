"""ROM archive format (rom_archive.cpp:65-190) and multi-source projection
(romgen.cpp:359-363, 446-455): Python writer/reader, the C++ mirror
(include/mswave/rom_archive.hpp, in libmswave_b200.so) byte for byte, the
reference's error checks, and projection of new sources / receivers through
the archived interface bases.  CPU only."""
import os
import shutil
import struct
import subprocess

import numpy as np
import pytest

from paper_1604_06750_b200._ffi import ConfigError
from paper_1604_06750_b200.archive import (archive_io, flat_from_archive, project_receivers,
                                           project_sources, read_rom_archive, system_from_archive,
                                           write_rom_archive)
from paper_1604_06750_b200.offline import RomOptions, build_regular
from paper_1604_06750_b200.rom import FlatSystem, system_receiver, system_sources

HERE = os.path.dirname(os.path.abspath(__file__))
TOOL = os.path.join(HERE, "cpp", "archive_tool")


@pytest.fixture(scope="module")
def built():
    opt = RomOptions(m=3, omega_max=4.0, epsilon_rel=1e-3, max_basis_per_interface=4)
    return build_regular([17, 17], 0.5, [2, 2], opt, (8, 4, 0), (8, 12, 0)), opt


@pytest.fixture(scope="module")
def archive_dir(built, tmp_path_factory):
    b, opt = built
    d = str(tmp_path_factory.mktemp("rom") / "archive")
    write_rom_archive(d, b.system.roms, b.basis, opt)
    return d


@pytest.fixture(scope="module")
def tool():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "archive_tool"], check=True)
    return TOOL


def _same(a, b):
    return np.asarray(a).shape == np.asarray(b).shape and np.asarray(a).tobytes() == np.asarray(b).tobytes()


def test_python_round_trip_bitwise(built, archive_dir):
    b, opt = built
    ar = read_rom_archive(archive_dir)
    assert ar.opt.m == opt.m and ar.opt.max_basis_per_interface == opt.max_basis_per_interface
    assert len(ar.roms) == len(b.system.roms)
    for r0, r1 in zip(b.system.roms, ar.roms):
        assert (r0.cell, r0.m, r0.ktilde, r0.shift) == (r1.cell, r1.m, r1.ktilde, r1.shift)
        assert list(r0.iface_ids) == list(r1.iface_ids)
        assert list(r0.iface_offsets) == list(r1.iface_offsets)
        for a, c in zip(list(r0.ladder) + list(r0.ladder_hat), list(r1.ladder) + list(r1.ladder_hat)):
            assert _same(np.asfortranarray(a), np.asfortranarray(c))
        for a, c in zip(r0.g_proj + r0.q_proj, r1.g_proj + r1.q_proj):
            assert _same(a, c)
    for f, S in enumerate(b.basis.S):
        assert _same(np.asfortranarray(S), np.asfortranarray(ar.basis.S[f]))


def test_container_layout(archive_dir):
    # rom_archive.cpp:84-99: magic, u64 cell/m/ktilde/n_ifaces, f64 shift
    with open(os.path.join(archive_dir, "cell_0000.bin"), "rb") as fh:
        data = fh.read()
    assert data[:8] == b"MSWROM1\x00"
    cell, m, kt, nif = struct.unpack_from("<QQQQ", data, 8)
    assert (cell, m) == (0, 3) and nif == 2 and kt > 0


def test_cpp_mirror_copies_byte_for_byte(archive_dir, tool, tmp_path):
    dst = str(tmp_path / "copy")
    out = subprocess.run([tool, "copy", archive_dir, dst], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    for name in sorted(os.listdir(archive_dir)):
        if name.endswith(".bin"):
            with open(os.path.join(archive_dir, name), "rb") as a, open(os.path.join(dst, name), "rb") as c:
                assert a.read() == c.read(), name
    # the C++-written manifest reads back to the same archive
    a0, a1 = read_rom_archive(archive_dir), read_rom_archive(dst)
    assert a0.opt == a1.opt and a0.basis.omega_max == a1.basis.omega_max and a0.basis.epsilon == a1.basis.epsilon


def test_cpp_mirror_reads_same_values(built, archive_dir, tool):
    out = subprocess.run([tool, "read", archive_dir], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    _, nc, nf, s = out.stdout.split()
    ar = read_rom_archive(archive_dir)
    total = 0.0
    for r in ar.roms:  # same summation order as archive_tool
        for L in list(r.ladder) + list(r.ladder_hat):
            for x in np.asfortranarray(L).ravel(order="F"):
                total += float(x)
    assert (int(nc), int(nf)) == (len(ar.roms), len(ar.basis.S))
    assert float(s) == total


def _corrupt(src, dst, fn):
    shutil.copytree(src, dst)
    fn(dst)
    return dst


@pytest.mark.parametrize("case,msg", [
    ("magic", "bad magic in ROM container"),
    ("truncated", "truncated ROM container"),
    ("basis", "mismatched interface bases between neighbor cells (interface"),
    ("manifest", "missing manifest.json in"),
    ("format", "not a ROM archive"),
])
def test_reference_error_checks(archive_dir, tool, tmp_path, case, msg):
    def magic(d):
        p = os.path.join(d, "cell_0001.bin")
        data = bytearray(open(p, "rb").read())
        data[0] = ord("X")
        open(p, "wb").write(bytes(data))

    def truncated(d):
        p = os.path.join(d, "cell_0002.bin")
        data = open(p, "rb").read()
        open(p, "wb").write(data[:len(data) // 2])

    def basis(d):
        # flip one bit of cell 1's copy of its first interface basis
        p = os.path.join(d, "cell_0001.bin")
        data = bytearray(open(p, "rb").read())
        off = 8 + 32 + 8 + 8 + 16  # header, shift, iface id, mat dims
        data[off] ^= 1
        open(p, "wb").write(bytes(data))

    def manifest(d):
        os.remove(os.path.join(d, "manifest.json"))

    def fmt(d):
        p = os.path.join(d, "manifest.json")
        text = open(p).read()
        open(p, "w").write(text.replace("mswave-rom-archive", "something-else"))

    d = _corrupt(archive_dir, str(tmp_path / case), {"magic": magic, "truncated": truncated, "basis": basis,
                                                     "manifest": manifest, "format": fmt}[case])
    with pytest.raises(ConfigError, match=msg.replace("(", r"\(")):
        read_rom_archive(d)
    out = subprocess.run([tool, "read", d], capture_output=True, text=True)
    assert out.returncode == 2 and out.stdout.startswith("error " + msg), out.stdout


def test_projection_reproduces_archived_io(built, archive_dir):
    # the ROMs were built with point source g and receiver q: projecting them
    # again through the archived S_f gives the archived g~ / q~ bit for bit
    b, _ = built
    ar = read_rom_archive(archive_dir)
    g_ar, rc_ar = archive_io(ar)
    G = project_sources(b.partition, ar.basis, [b.g])
    assert _same(G, g_ar)
    rc = project_receivers(b.partition, ar.basis, [b.q])
    assert np.array_equal(rc.term_iface, rc_ar.term_iface) and _same(rc.term_q, rc_ar.term_q)
    # sparse (rows, values) form is the same
    nz = np.nonzero(b.g)[0]
    assert _same(project_sources(b.partition, ar.basis, [(nz, b.g[nz])]), G)
    # and equals what assemble_system hands the stepper
    assert _same(G, system_sources(b.system))


def test_multi_source_projection_and_skeleton_check(built, archive_dir):
    b, _ = built
    ar = read_rom_archive(archive_dir)
    part = b.partition
    sk = np.asarray(part.skeleton)
    rng = np.random.default_rng(5)
    picks = rng.choice(sk, size=6, replace=False)
    srcs = [(np.array([k]), np.array([1.0])) for k in picks]
    G = project_sources(part, ar.basis, srcs)
    assert G.shape == (flat_from_archive(ar).total_io, 6)
    for s, k in enumerate(picks):  # column s = rows of S_f at node k, for every interface holding k
        expect = np.zeros(G.shape[0])
        off = 0
        for f, I in enumerate(part.interfaces):
            Mf = ar.basis.S[f].shape[1]
            pos = np.searchsorted(I.nodes, k)
            if pos < len(I.nodes) and I.nodes[pos] == k:
                expect[off:off + Mf] = ar.basis.S[f][pos, :]
            off += Mf
        assert _same(G[:, s], expect)
    interior = np.setdiff1d(np.arange(part.n_nodes), sk)[0]
    with pytest.raises(ConfigError, match="source has support off the partition skeleton"):
        project_sources(part, ar.basis, [(np.array([interior]), np.array([1.0]))])
    with pytest.raises(ConfigError, match="receiver has support off the partition skeleton"):
        project_receivers(part, ar.basis, [(np.array([interior]), np.array([1.0]))])


def test_system_from_archive_matches_original(built, archive_dir):
    b, _ = built
    ar = read_rom_archive(archive_dir)
    sys2 = system_from_archive(b.partition, ar, b.pencil.B)
    f0, f1 = FlatSystem.from_system(b.system), FlatSystem.from_system(sys2)
    for k in ("cell_m", "cell_ktilde", "cell_iface_ptr", "cell_iface_ids", "cell_iface_offsets",
              "cell_ladder_off", "ladders", "iface_ci", "iface_cj", "iface_li", "iface_lj", "iface_size"):
        assert _same(getattr(f0, k), getattr(f1, k)), k
    for i0, i1 in zip(b.system.ifaces, sys2.ifaces):
        assert _same(i0.mass, i1.mass)
    # topology straight from the archive (no partition) agrees as well
    fa = flat_from_archive(ar)
    for k in ("cell_iface_ids", "cell_iface_offsets", "ladders", "iface_ci", "iface_cj", "iface_li",
              "iface_lj", "iface_size"):
        assert _same(getattr(f0, k), getattr(fa, k)), k
    with pytest.raises(ConfigError, match="cell count does not match"):
        from paper_1604_06750_b200.archive import RomArchive
        system_from_archive(b.partition, RomArchive(ar.roms[:-1], ar.basis, ar.opt), b.pencil.B)


def test_c_abi_archive_errors_without_device(tmp_path):
    # msw_create_from_archive reports the reader's ConfigError (code 2, the
    # reference's message) before any device work
    import ctypes as C

    from paper_1604_06750_b200 import _ffi
    lib = _ffi.load()
    h = C.c_void_p()
    rc = lib.msw_create_from_archive(str(tmp_path / "nope").encode(), 0, C.byref(h))
    assert rc == _ffi.MSW_CONFIG_ERROR
    assert lib.msw_last_error().decode().startswith("missing manifest.json in")
    (tmp_path / "bad").mkdir()
    (tmp_path / "bad" / "manifest.json").write_text('{"format": "something-else"}')
    rc = lib.msw_create_from_archive(str(tmp_path / "bad").encode(), 0, C.byref(h))
    assert rc == _ffi.MSW_CONFIG_ERROR and "not a ROM archive" in lib.msw_last_error().decode()
    (tmp_path / "bad" / "manifest.json").write_text('{"format": "mswave-rom-archive", "m": 2,')
    rc = lib.msw_create_from_archive(str(tmp_path / "bad").encode(), 0, C.byref(h))
    assert rc == _ffi.MSW_CONFIG_ERROR and "malformed JSON" in lib.msw_last_error().decode()
