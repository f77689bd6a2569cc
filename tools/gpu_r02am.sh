#!/bin/bash
o=gpurun_out/am; mkdir -p $o
timeout 1200 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "every_k1_kernel_family" > $o/family.log 2>&1; tail -2 $o/family.log
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 50 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
nrun c5:128 MSW_K1_VARIANT=105
nrun c5:128 MSW_K1_VARIANT=105 MSW_K1_NP=32
nrun c5:128 MSW_K1_VARIANT=95
nrun c5:128 MSW_K1_VARIANT=95 MSW_K1_ST=64
