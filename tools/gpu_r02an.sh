#!/bin/bash
# K2 (rom_iface_step) threads per CTA A/B
o=gpurun_out/an; mkdir -p $o
export MSW_TUNE_CACHE=$PWD/$o/tune_cache.txt
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 100 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'])
"; }
for t in 128 64 96 192 256; do nrun c3:64,c5:32,c5:128,c5:8 MSW_K2_THREADS=$t; done
