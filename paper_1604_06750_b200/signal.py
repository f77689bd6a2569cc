"""Source signature (proj/include/mswave/wavelet.hpp, proj/src/wavelet.cpp).

``Wavelet.__call__`` restates wavelet.cpp:9-19 with libm ``exp`` (Python's
math.exp), so samples are bit-identical to the C++ reference and oracle.
The Ricker kind is an extension (absent from the reference, wavelet.hpp:12):
(1 - x^2) exp(-x^2/2) with the same x = (t - t0)/tau; with the default
width_factor 3.5 its peak frequency is omega_cut / (3.5 sqrt(2) pi), i.e.
f_max = omega_cut/2pi ~ 2.5 f_peak.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._ffi import ConfigError

KINDS = ("gaussian_derivative", "gaussian", "ricker")


@dataclass
class Wavelet:
    kind: str = "gaussian_derivative"
    omega_cut: float = 2.0 * 3.14159265358979323846
    width_factor: float = 3.5
    delay_factor: float = 6.0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ConfigError(f"unknown wavelet kind: {self.kind}")

    @property
    def kind_id(self) -> int:
        return KINDS.index(self.kind)

    def tau(self) -> float:
        return self.width_factor / self.omega_cut

    def delay(self) -> float:
        return self.delay_factor * self.tau()

    def __call__(self, t: float) -> float:
        x = (t - self.delay()) / self.tau()
        if self.kind == "gaussian_derivative":
            return -x * math.exp(0.5 - 0.5 * x * x)
        if self.kind == "gaussian":
            return math.exp(-0.5 * x * x)
        return (1.0 - x * x) * math.exp(-0.5 * x * x)

    def samples_accumulated(self, dt: float, steps: int, t0: float = 0.0):
        """ROM time base: w(st.t) with st.t accumulated (msolver.cpp:191,415).
        Returns (w[steps], times[steps+1])."""
        w = np.empty(steps)
        times = np.empty(steps + 1)
        t = t0
        times[0] = t
        for n in range(steps):
            w[n] = self(t)
            t += dt
            times[n + 1] = t
        return w, times

    def samples_fixed(self, dt: float, steps: int):
        """Fine time base: t_s = s*dt (reference.cpp:67).  Returns
        (w[steps], times[steps+1])."""
        w = np.array([self(float(s) * dt) for s in range(steps)])
        times = np.array([float(s) * dt for s in range(steps + 1)])
        return w, times


def steps_for(t_final: float, dt: float) -> int:
    """steps = ceil(t_final/dt - 1e-12) (msolver.cpp:401, reference.cpp:55)."""
    return int(math.ceil(t_final / dt - 1e-12))
