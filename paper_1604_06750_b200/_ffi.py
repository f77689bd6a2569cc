"""ctypes binding of the product C ABI (include/mswave_b200.h).

The shared library ``libmswave_b200.so`` (CUDA kernels for sm_100a + the C
ABI) is built in-tree by ``__graft_entry__.build()`` / ``make -C
paper_1604_06750_b200/csrc``.  There is no CPU fallback: if the library is
missing, importing the stepper raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MSW_LIB: load another build of the library (A/B timing of kernel changes)
LIB_PATH = os.environ.get("MSW_LIB", os.path.join(_HERE, "libmswave_b200.so"))

ABI_VERSION = 3  # MSW_ABI_VERSION of include/mswave_b200.h
MSW_OK = 0
MSW_CONFIG_ERROR = 2
MSW_NUMERICAL_ERROR = 3
MSW_CUDA_ERROR = 4

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class ConfigError(RuntimeError):
    """mirror of mswave::ConfigError (types.hpp:31-34), exit code 2"""


class NumericalError(RuntimeError):
    """mirror of mswave::NumericalError (types.hpp:25-29), exit code 3"""


class CudaError(RuntimeError):
    """device / runtime failure (no reference analogue)"""


class SystemDesc(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int32),
        ("n_ifaces", C.c_int32),
        ("cell_m", i32p),
        ("cell_ktilde", i32p),
        ("cell_iface_ptr", i32p),
        ("cell_iface_ids", i32p),
        ("cell_iface_offsets", i32p),
        ("cell_ladder_off", i64p),
        ("ladders", f64p),
        ("iface_ci", i32p),
        ("iface_cj", i32p),
        ("iface_li", i32p),
        ("iface_lj", i32p),
        ("iface_size", i32p),
        ("iface_mass", f64p),
    ]


class Info(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int64),
        ("n_ifaces", C.c_int64),
        ("n_flat", C.c_int64),
        ("reduced_dof", C.c_int64),
        ("flops_per_step", C.c_int64),
        ("dense_entries", C.c_int64),
        ("sources", C.c_int64),
        ("receivers", C.c_int64),
        ("device_bytes", C.c_int64),
        ("k1_variant", C.c_int64),
        ("k1_source_tile", C.c_int64),
        ("k1_panel", C.c_int64),
        ("k1_rings", C.c_int64),
        ("k1_tune_cached", C.c_int64),
        ("k1_fuse_kappa", C.c_double),
    ]


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


_PROTOS = {
    "msw_abi_version": (C.c_int, []),
    "msw_last_error": (C.c_char_p, []),
    "msw_create": (C.c_int, [C.POINTER(SystemDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "msw_create_from_archive": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "msw_estimate_dt": (C.c_int, [C.c_void_p, C.c_double, f64p]),
    "msw_energy": (C.c_int, [C.c_void_p, f64p]),
    "msw_destroy": (None, [C.c_void_p]),
    "msw_get_info": (C.c_int, [C.c_void_p, C.POINTER(Info)]),
    "msw_get_masses": (C.c_int, [C.c_void_p, f64p, f64p]),
    "msw_set_sources": (C.c_int, [C.c_void_p, C.c_int32, f64p]),
    "msw_set_receivers": (C.c_int, [C.c_void_p, C.c_int32, i32p, i32p, f64p]),
    "msw_set_corners": (C.c_int, [C.c_void_p, C.c_int32, i32p, i32p, i32p, f64p, i32p, f64p]),
    "msw_make_state": (C.c_int, [C.c_void_p, C.c_double]),
    "msw_step": (C.c_int, [C.c_void_p, f64p, C.c_int32]),
    "msw_corner_correct": (C.c_int, [C.c_void_p]),
    "msw_get_state": (C.c_int, [C.c_void_p, f64p, f64p, f64p, f64p, f64p, i64p]),
    "msw_set_state": (C.c_int, [C.c_void_p, f64p, f64p, f64p, f64p, C.c_double, C.c_int64]),
    "msw_run": (C.c_int, [C.c_void_p, C.c_int64, f64p, C.c_int32, C.c_int32, f64p, f64p, i64p]),
    "msw_run_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32,
                                 C.c_void_p, C.c_void_p]),
    "msw_check_instability": (C.c_int, [C.c_void_p, i64p]),
    "msw_prepare": (C.c_int, [C.c_void_p, C.c_int32]),
    "msw_last_launch_count": (C.c_int, [C.c_void_p, i64p]),
    "msw_time_kernels": (C.c_int, [C.c_void_p, C.c_int32, f64p]),
    "msw_fine_create": (C.c_int, [C.c_int32, i32p, C.c_double, f64p, f64p, C.c_int,
                                  C.POINTER(C.c_void_p)]),
    "msw_fine_destroy": (None, [C.c_void_p]),
    "msw_fine_size": (C.c_int, [C.c_void_p, i64p]),
    "msw_fine_leapfrog": (C.c_int, [C.c_void_p, C.c_int32, i32p, i64p, f64p, C.c_int32, i32p,
                                    i64p, f64p, C.c_double, C.c_int64, f64p, C.c_int32, f64p,
                                    i64p]),
    "msw_fine_leapfrog_device": (C.c_int, [C.c_void_p, C.c_int32, i32p, i64p, f64p, C.c_int32,
                                           i32p, i64p, f64p, C.c_double, C.c_int64, C.c_void_p,
                                           C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "msw_fine_check_instability": (C.c_int, [C.c_void_p, i64p]),
    "msw_fine_create_csc": (C.c_int, [C.c_int64, i32p, i32p, f64p, f64p, C.c_int, C.POINTER(C.c_void_p)]),
    "msw_fine_cfl": (C.c_int, [C.c_void_p, f64p]),
}

EXPORTED_SYMBOLS = tuple(_PROTOS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the product library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(path)
    lib.msw_abi_version.restype = C.c_int
    if lib.msw_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI version {lib.msw_abi_version()}, expected {ABI_VERSION} (rebuild)")
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, lib=None):
    if rc == MSW_OK:
        return
    lib = lib or load()
    msg = lib.msw_last_error().decode()
    if rc == MSW_CONFIG_ERROR:
        raise ConfigError(msg)
    if rc == MSW_NUMERICAL_ERROR:
        raise NumericalError(msg)
    raise CudaError(msg)
