#!/bin/bash
# two-CTA-per-SM K-streaming instances (89-93): parity, then config 5 S = 32 / 128
o=gpurun_out/ac; mkdir -p $o
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "every_k1_kernel_family" > $o/family.log 2>&1; tail -3 $o/family.log
for v in 89 90 91 92 93; do
  MSW_K1_VARIANT=$v MSW_K1_TUNE_LOG=1 timeout 600 python tools/rom_sweep.py --cases c5:32,c5:128 --steps 30 > $o/v$v.log 2> $o/v$v.tune
  python - <<PY
import json
for l in open("$o/v$v.log"):
    try:
        d = json.loads(l); print($v, d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], {k:v for k,v in d['k1'].items() if k!='k1_variant'})
    except Exception as e: print('ERR', l[:200])
PY
done
