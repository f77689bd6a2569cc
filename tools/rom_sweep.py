"""Quick device-time sweep of the on-line ROM step over BASELINE configs
(development aid; bench.py is the contract).  Prints one JSON line per
(config, S): ms/step (CUDA events over K steps on a dedicated stream),
per-kernel ms (K1 / K2 timed alone), algorithmic GB/s and TF/s."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_06750_b200.rom import RomStepper  # noqa: E402
from paper_1604_06750_b200.synthetic import config_case  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="c3:64,c5:1,c5:8,c5:32,c5:128")
ap.add_argument("--steps", type=int, default=100)
args = ap.parse_args()
PEAK, _ = bench.load_peaks()
ts = torch.cuda.Stream()
torch.cuda.set_stream(ts)
for spec in args.cases.split(","):
    cfg, S = spec.split(":")
    S = int(S)
    case = config_case(cfg, S=S)
    st = RomStepper(case.flat)
    st.set_sources(case.g)
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    K = args.steps
    w = torch.ones(K + 10, dtype=torch.float64, device="cuda")
    tr = torch.empty((K + 1) * st.R * S, dtype=torch.float64, device="cuda")
    st.prepare()
    st.run_device(5, w.data_ptr(), 1, tr.data_ptr(), ts.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.run_device(K, w.data_ptr(), 1, tr.data_ptr(), ts.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    bad = st.check_instability()
    st.make_state(case.dt)
    k1, k2 = st.time_kernels(20)
    b1, f1 = bench.cell_kernel_bytes(case.flat, S)
    sb = bench.step_bytes(case.flat, S)
    print(json.dumps({"config": cfg, "S": S, "ms_step": ms, "k1_ms": k1, "k2_ms": k2,
                      "step_gbs": sb / ms / 1e6, "step_frac": sb / ms / 1e6 / PEAK,
                      "k1_gbs": b1 / k1 / 1e6, "k1_frac": b1 / k1 / 1e6 / PEAK,
                      "k1_tflops": f1 / k1 / 1e9, "unstable": bad,
                      "dof_upd_s": case.flat.n_flat * S / (ms / 1e3),
                      "k1": {k: v for k, v in st.info().items() if k.startswith("k1_")}}), flush=True)
    del st, w, tr
    torch.cuda.empty_cache()
