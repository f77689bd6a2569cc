#!/bin/bash
o=gpurun_out/s10; mkdir -p $o
timeout 1500 python -m pytest tests/test_rom_gpu.py -x -q -m gpu > $o/rom_tests.log 2>&1
tail -2 $o/rom_tests.log
for dbg in 0 1; do
echo "== dbg $dbg" >> $o/c5.log
MSW_K1_DEBUG=$dbg timeout 600 python tools/rom_sweep.py --cases c5:32,c5:128 --steps 50 2>&1 | cut -c1-700 >> $o/c5.log
done
python - <<'PY'
import json
for l in open("gpurun_out/s10/c5.log"):
    if l.startswith('=='): print(l.strip()[:70])
    else:
        try:
            d = json.loads(l); print(d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1'])
        except Exception as e: print('ERR', l[:100])
PY
