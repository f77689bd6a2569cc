"""Every BASELINE.json configuration the bench or README reports, run at its
own configured shape through the autotuned kernel instance it runs in the
bench, against the oracle restatement of the reference's stepper
(msolver.cpp:154-194, 397-424): receiver traces within relative L2 1e-10 (the
north-star gate) per (receiver, source) trace.

  config 1: 8^3 cells, M = 1, S = 1, the full 2000 steps;
  config 2: 8^3 cells of 16, M = 6, all 16 sources, the full 3000 steps;
  config 3: 16^3 cells, M = 6, S = 64 on the GPU, 4 of the sources through
            the oracle over the full 4000 steps (slow: ~3 min of oracle time);
  config 5: 16^3 cells of 24, M = 17, S = 1 / 8 / 32 / 128 on the GPU, 1-2
            sources through the oracle over 100 steps.

Each test also asserts the tuner's pick is an instance covered by the
bitwise family tests of tests/test_rom_gpu.py (TESTED_VARIANTS)."""
import os
import time

import numpy as np
import pytest

from paper_1604_06750_b200.rom import RomStepper
from paper_1604_06750_b200.signal import Wavelet
from paper_1604_06750_b200.synthetic import config_case
from tests.helpers import per_trace_rel_l2
from tests.test_rom_gpu import TESTED_VARIANTS

pytestmark = pytest.mark.gpu
TOL = 1e-10
THREADS = max(1, min(16, os.cpu_count() or 1))


def _run_case(oracle, name, S, steps, n_oracle, second_handle=False):
    case = config_case(name, S=S)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, steps)
    st = RomStepper(case.flat)
    st.set_sources(case.g)
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    info = st.info()
    tg, times = st.run(steps, w)
    st.close()
    ora = oracle.OracleStepper(case.flat)
    ora.set_sources(np.ascontiguousarray(case.g[:, :n_oracle]))
    ora.set_receivers(case.receivers)
    ora.make_state(case.dt)
    to, tio = ora.run(steps, w, threads=min(THREADS, n_oracle))
    assert np.array_equal(times, tio)
    assert np.abs(to).max() > 0
    err = per_trace_rel_l2(tg[:, :, :n_oracle], to)
    assert err < TOL, (name, S, err, info)
    assert info["k1_variant"] in TESTED_VARIANTS, info
    if second_handle:
        # the tuning cache: a second system of the same shape reuses the
        # first one's geometry without re-timing, and its bits are the same
        st2 = RomStepper(case.flat)
        st2.set_sources(case.g)
        st2.set_receivers(case.receivers)
        t0 = time.perf_counter()
        st2.make_state(case.dt)
        t_make = time.perf_counter() - t0
        info2 = st2.info()
        tg2, _ = st2.run(steps, w)
        st2.close()
        assert info2["k1_tune_cached"] == 1 and info2["k1_variant"] == info["k1_variant"], (info, info2)
        assert t_make < 0.5, t_make
        assert np.array_equal(tg2, tg)
    return info


def test_config1_full_length(gpu_lib, oracle):
    _run_case(oracle, "c1", 1, 2000, 1)


def test_config2_full_length_all_sources(gpu_lib, oracle):
    _run_case(oracle, "c2", 16, 3000, 16)


@pytest.mark.slow
def test_config3_full_length_source_subset(gpu_lib, oracle):
    _run_case(oracle, "c3", 64, 4000, 4)


@pytest.mark.parametrize("S,n_oracle", [(1, 1), (8, 1), (32, 2), (128, 2)])
def test_config5_sweep_points(gpu_lib, oracle, S, n_oracle):
    _run_case(oracle, "c5", S, 100, n_oracle, second_handle=S == 32)


def test_tuning_cache_file_across_processes(gpu_lib, tmp_path):
    """MSW_TUNE_CACHE: a second process tuning the same shape reuses the
    first process's geometry from the file (msw_info.k1_tune_cached)."""
    import json
    import subprocess
    import sys

    code = ("import json, sys; sys.path.insert(0, %r)\n"
            "from paper_1604_06750_b200.rom import RomStepper\n"
            "from paper_1604_06750_b200.synthetic import config_case\n"
            "case = config_case('c5', S=8)\n"
            "st = RomStepper(case.flat); st.set_sources(case.g); st.set_receivers(case.receivers)\n"
            "st.make_state(case.dt); print(json.dumps(st.info()))\n") % os.path.dirname(os.path.dirname(__file__))
    env = dict(os.environ, MSW_TUNE_CACHE=str(tmp_path / "tune.txt"))
    env.pop("MSW_K1_VARIANT", None)
    infos = []
    for _ in range(2):
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr
        infos.append(json.loads(out.stdout.strip().splitlines()[-1]))
    assert infos[0]["k1_tune_cached"] == 0 and infos[1]["k1_tune_cached"] == 1
    assert infos[0]["k1_variant"] == infos[1]["k1_variant"] and infos[0]["k1_rings"] == infos[1]["k1_rings"]
    assert (tmp_path / "tune.txt").read_text().count("\n") >= 1
