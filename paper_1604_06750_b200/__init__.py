"""B200-native on-line stage of the multiscale S-fraction ROM wave solver
(arXiv 1604.06750): hand-written sm_100a fp64 kernels behind the C ABI of
include/mswave_b200.h, with a Python mirror of the reference's
proj/include/mswave API for tests and benchmarks.

The CUDA library is mandatory: there is no CPU fallback.  ``RomStepper`` /
``FineGrid`` raise ImportError if ``libmswave_b200.so`` has not been built.
"""
from ._ffi import ConfigError, CudaError, NumericalError, LIB_PATH, load  # noqa: F401
from .rom import (CornerCopy, CornerGroup, CoupledInterface, FlatSystem,  # noqa: F401
                  MultiscaleSystem, Receivers, RomStepper, SubdomainROM)
from .signal import Wavelet, steps_for  # noqa: F401
from .fine import FineGrid, GridMedium, make_uniform_medium  # noqa: F401

__all__ = [
    "ConfigError", "NumericalError", "CudaError", "load", "LIB_PATH",
    "SubdomainROM", "CoupledInterface", "CornerCopy", "CornerGroup", "MultiscaleSystem",
    "FlatSystem", "Receivers", "RomStepper", "Wavelet", "steps_for", "FineGrid", "GridMedium",
    "make_uniform_medium",
]
