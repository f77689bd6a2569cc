"""The product's compare_traces (paper_1604_06750_b200/traces.py) against the
oracle restatement of trace_io.cpp:36-67: resampling, truncation at the
shorter trace, the zero-reference fallback."""
import numpy as np
import pytest

from paper_1604_06750_b200._ffi import ConfigError
from paper_1604_06750_b200.traces import compare_traces


@pytest.mark.parametrize("na,nb,dta,dtb", [(101, 101, 0.1, 0.1), (201, 97, 0.05, 0.11), (50, 400, 0.3, 0.02)])
def test_compare_traces_matches_oracle(oracle, na, nb, dta, dtb):
    rng = np.random.default_rng(na + nb)
    at = np.arange(na) * dta
    bt = np.arange(nb) * dtb
    av = np.sin(1.3 * at) + 0.01 * rng.standard_normal(na)
    bv = np.sin(1.3 * bt)
    mx, rl = oracle.compare_traces(at, av, bt, bv)
    rep = compare_traces(at, av, bt, bv)
    assert rep["max_abs_error"] == pytest.approx(mx, rel=1e-12, abs=1e-15)
    assert rep["rel_l2_error"] == pytest.approx(rl, rel=1e-12)


def test_compare_traces_zero_reference_and_empty(oracle):
    t = np.arange(10) * 0.5
    a = np.linspace(0, 1, 10)
    z = np.zeros(10)
    mx, rl = oracle.compare_traces(t, a, t, z)
    rep = compare_traces(t, a, t, z)
    assert rep["rel_l2_error"] == pytest.approx(rl, rel=1e-12)
    assert rep["rel_l2_error"] == pytest.approx(np.sqrt(np.sum(a * a)), rel=1e-12)
    with pytest.raises(ConfigError, match="cannot compare empty traces"):
        compare_traces([], [], t, z)
