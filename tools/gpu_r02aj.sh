#!/bin/bash
# live-tile dispatch in the fused stage form: parity, config 1-3 timing
o=gpurun_out/aj; mkdir -p $o
timeout 1200 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "fused" > $o/rom.log 2>&1; tail -3 $o/rom.log
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 200 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
nrun c3:64 MSW_K1_VARIANT=86
nrun c3:64 MSW_K1_VARIANT=69
nrun c3:64,c3:1,c3:16,c2:16,c1:1
