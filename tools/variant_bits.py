"""Bitwise comparison of K1 instances on a BASELINE config (development aid):
runs the same case for --steps steps under each MSW_K1_VARIANT in --variants
and reports whether traces and final states are identical to the first."""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_06750_b200.rom import RomStepper  # noqa: E402
from paper_1604_06750_b200.signal import Wavelet  # noqa: E402
from paper_1604_06750_b200.synthetic import config_case  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--S", type=int, default=64)
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--variants", default="69,86")
args = ap.parse_args()
case = config_case(args.config, S=args.S)
w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, args.steps)
ref = None
for v in args.variants.split(","):
    os.environ["MSW_K1_VARIANT"] = v
    st = RomStepper(case.flat)
    st.set_sources(case.g)
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    tr, _ = st.run(args.steps, w)
    u = st.get_state()["u_cur"]
    got = int(st.info()["k1_variant"])
    if ref is None:
        ref = (tr, u)
        same = None
    else:
        same = bool(np.array_equal(tr, ref[0]) and np.array_equal(u, ref[1]))
    digest = hashlib.sha256(np.ascontiguousarray(tr).tobytes() + np.ascontiguousarray(u).tobytes()).hexdigest()[:16]
    print(json.dumps({"variant": v, "ran": got, "bitwise_equal_first": same, "sha": digest,
                      "trace_absmax": float(np.abs(tr).max())}), flush=True)
    del st
