#!/bin/bash
o=gpurun_out/s5; mkdir -p $o
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "fused" > $o/fused_tests.log 2>&1
tail -3 $o/fused_tests.log
timeout 300 python tools/variant_bits.py --config c3 --S 64 --steps 64 --variants 69,86,89,90,91,92 > $o/bits.txt 2>&1
cat $o/bits.txt
for v in 86 89 92 90; do
  for rings in 6,4 7,3 7,4 6,3; do
    echo "== v $v rings $rings" >> $o/bs_sweep.log
    MSW_K1_VARIANT=$v MSW_K1_ST=64 MSW_K1_NP=40 MSW_K1_RINGS=$rings timeout 300 python tools/rom_sweep.py --cases c3:64 --steps 200 >> $o/bs_sweep.log 2>&1
  done
done
python - <<'PY'
import json
for f in ("gpurun_out/s5/bs_sweep.log",):
    for l in open(f):
        if l.startswith('=='): print(l.strip()[:60], end=' ')
        else:
            try:
                d = json.loads(l); print(round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_rings'])
            except Exception as e: print('ERR', l[:100])
PY
