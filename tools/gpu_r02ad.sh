#!/bin/bash
# two-CTA K-streaming instance 89: ring / chunk sweep and cycle breakdown
o=gpurun_out/ad; mkdir -p $o
run() { env "$@" MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=8 timeout 300 python tools/rom_sweep.py --cases c5:128 --steps 30 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'k1_prof' in d:
        p = d['k1_prof']; t = sum(p); print('   prof', [round(100*x/t,1) for x in p])
    else: print('$*', round(d['ms_step'],4), round(d['k1_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
run MSW_K1_VARIANT=89
run MSW_K1_VARIANT=89 MSW_K1_NP=8 MSW_K1_RINGS=4,4
run MSW_K1_VARIANT=89 MSW_K1_NP=8 MSW_K1_RINGS=6,3
run MSW_K1_VARIANT=91
run MSW_K1_VARIANT=91 MSW_K1_NP=8 MSW_K1_RINGS=4,4
run MSW_K1_VARIANT=90
run MSW_K1_VARIANT=90 MSW_K1_NP=16 MSW_K1_RINGS=3,3
run MSW_K1_VARIANT=42
