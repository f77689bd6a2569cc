#!/bin/bash
o=gpurun_out/s9; mkdir -p $o
for h in 1 0 3 2 1 3; do
echo "== l2hint $h" >> $o/l2.log
MSW_L2HINT=$h MSW_K1_VARIANT=86 MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=6,4 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 2>&1 >> $o/l2.log
done
MSW_K1_TUNE_LOG=1 MSW_TUNE_FRESH=1 timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 > $o/tune.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/s9/l2.log"):
    if l.startswith('=='): print(l.strip()[:70], end=' ')
    else:
        try:
            d = json.loads(l); print(round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_rings'])
        except Exception as e: print('ERR', l[:100])
PY
grep k1_tune gpurun_out/s9/tune.log | sort -t: -k7 | cut -c1-120 | head -50
tail -1 gpurun_out/s9/tune.log | cut -c1-300
