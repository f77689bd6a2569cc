"""Development probe for rom_cell_fused on small shapes (python tools/fused_probe.py VARIANT m cells M S)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_1604_06750_b200.rom import RomStepper  # noqa: E402
from paper_1604_06750_b200.signal import Wavelet  # noqa: E402
from paper_1604_06750_b200.synthetic import synthetic_system  # noqa: E402

os.environ["MSW_K1_FUSED"] = "1"
os.environ["MSW_K1_VARIANT"] = sys.argv[1]
m = int(sys.argv[2])
cells = tuple(int(x) for x in sys.argv[3].split("x"))
M, S = int(sys.argv[4]), int(sys.argv[5])
case = synthetic_system(cells, M=M, m=m, S=S, R=2, seed=3)
g = RomStepper(case.flat)
g.set_sources(case.g)
g.set_receivers(case.receivers)
g.make_state(case.dt)
print("info", {k: v for k, v in g.info().items() if k.startswith("k1")}, flush=True)
w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, 3)
t, _ = g.run(3, w)
print("ok", float(np.abs(t).max()), flush=True)
