"""e2e (msw_run, pinned host buffers) vs device time at config 3 (development aid)."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_06750_b200.rom import RomStepper
from paper_1604_06750_b200.synthetic import config_case
from paper_1604_06750_b200.signal import Wavelet
cfg, S = (sys.argv[1] if len(sys.argv) > 1 else "c3:64").split(":")
case = config_case(cfg, S=int(S))
st = RomStepper(case.flat); st.set_sources(case.g); st.set_receivers(case.receivers); st.make_state(case.dt)
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, K)
w_pin = torch.tensor(w, dtype=torch.float64).pin_memory()
tr = torch.empty((K + 1, st.R, st.S), dtype=torch.float64).pin_memory()
tm = torch.empty(K + 1, dtype=torch.float64).pin_memory()
for rep in range(4):
    st.make_state(case.dt); st.prepare()
    t0 = time.perf_counter(); st.run(K, w_pin.numpy(), traces_out=tr.numpy(), times_out=tm.numpy()); t = time.perf_counter() - t0
    print(json.dumps({"case": sys.argv[1:] , "overlap": os.environ.get("MSW_RUN_OVERLAP", "1"), "pdl": os.environ.get("MSW_PDL", "1"), "rep": rep, "ms_per_step": 1e3 * t / K}), flush=True)
