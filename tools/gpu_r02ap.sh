#!/bin/bash
# K2: pre-barrier operand loads (HOIST) on / off at 96 and 64 threads
o=gpurun_out/ap; mkdir -p $o
export MSW_TUNE_CACHE=$PWD/$o/tune_cache.txt
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 100 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'])
"; }
nrun c3:64,c5:32,c5:128,c5:8 X=0
nrun c3:64,c5:32,c5:128,c5:8 MSW_K2_HOIST=1
nrun c3:64,c5:32,c5:128,c5:8 MSW_K2_HOIST=0
nrun c3:64,c5:32,c5:128,c5:8 MSW_K2_HOIST=1 MSW_K2_THREADS=64
nrun c3:64,c5:32,c5:128,c5:8 MSW_K2_THREADS=32
