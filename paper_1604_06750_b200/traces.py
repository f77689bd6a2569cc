"""compare_traces (trace_io.cpp:36-67): max-abs and relative-L2 error of
trace a against trace b, b linearly resampled onto a's times (samples past
the shorter trace's end are ignored; relative L2 falls back to absolute when
b is identically zero).  Host-side helper of the public API (the C++ mirror
has the same function, include/mswave/trace_io.hpp)."""
from __future__ import annotations

import numpy as np

from ._ffi import ConfigError


def compare_traces(a_times, a_values, b_times, b_values) -> dict:
    at = np.asarray(a_times, np.float64)
    av = np.asarray(a_values, np.float64)
    bt = np.asarray(b_times, np.float64)
    bv = np.asarray(b_values, np.float64)
    if at.size == 0 or bt.size == 0:
        raise ConfigError("cannot compare empty traces")
    t_end = min(at[-1], bt[-1])
    keep = at <= t_end + 1e-12
    # a stops at the first sample past t_end (the reference breaks there)
    stop = int(np.argmin(keep)) if not keep.all() else at.size
    t = at[:stop]
    hi = np.searchsorted(bt, t, side="right")
    hi = np.clip(hi, 1, bt.size - 1)
    lo = hi - 1
    with np.errstate(invalid="ignore", divide="ignore"):
        w = (t - bt[lo]) / (bt[hi] - bt[lo])
    samp = (1.0 - w) * bv[lo] + w * bv[hi]
    samp = np.where(t <= bt[0], bv[0], np.where(t >= bt[-1], bv[-1], samp))
    d = av[:stop] - samp
    num2 = float(np.sum(d * d))
    den2 = float(np.sum(samp * samp))
    return {"max_abs_error": float(np.max(np.abs(d))) if d.size else 0.0,
            "rel_l2_error": float(np.sqrt(num2 / den2)) if den2 > 0.0 else float(np.sqrt(num2)),
            "steps_a": int(at.size - 1), "steps_b": int(bt.size - 1),
            "dt_a": float(at[1] - at[0]) if at.size > 1 else 0.0,
            "dt_b": float(bt[1] - bt[0]) if bt.size > 1 else 0.0}
