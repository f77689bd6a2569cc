"""Real config-2 ROM (data/rom_c2): traces of each K1 numerical family against
the oracle (development aid for the family rule)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle_ffi  # noqa: E402
from paper_1604_06750_b200.archive import flat_from_archive, read_rom_archive  # noqa: E402
from paper_1604_06750_b200.rom import Receivers, RomStepper  # noqa: E402
from paper_1604_06750_b200.signal import Wavelet  # noqa: E402
from tests.helpers import per_trace_rel_l2  # noqa: E402

arch = os.path.join(ROOT, "data", "rom_c2")
io = np.load(os.path.join(arch, "io.npz"))
rc = Receivers(io["rcv_ptr"].astype(np.int32), io["rcv_iface"].astype(np.int32), io["rcv_q"])
flat = flat_from_archive(read_rom_archive(arch))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
o = oracle_ffi.OracleStepper(flat)
o.set_sources(np.ascontiguousarray(io["g"]))
o.set_receivers(rc)
dt = 0.9 * o.estimate_dt(1.0) * 0.5
w, _ = Wavelet(kind="ricker", omega_cut=float(io["omega_max"])).samples_accumulated(dt, steps)
o.make_state(dt)
to, _ = o.run(steps, w, threads=os.cpu_count() or 1)
for env in ({"MSW_K1_FUSED": "0"}, {"MSW_K1_FUSED": "1"}, {"MSW_K1_FUSED": "0", "MSW_K1_VARIANT": "4"}):
    for k in ("MSW_K1_FUSED", "MSW_K1_VARIANT"):
        os.environ.pop(k, None)
    os.environ.update(env)
    st = RomStepper(flat)
    st.set_sources(io["g"])
    st.set_receivers(rc)
    st.make_state(dt)
    tg, _ = st.run(steps, w)
    info = st.info()
    st.close()
    print(json.dumps({"env": env, "k1_variant": info["k1_variant"], "rel_l2_vs_oracle": per_trace_rel_l2(tg, to),
                      "steps": steps}), flush=True)
