#!/bin/bash
o=gpurun_out/ah; mkdir -p $o
run() { cases=$1; shift; env "$@" MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=8 timeout 300 python tools/rom_sweep.py --cases $cases --steps 100 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'k1_prof' in d:
        p = d['k1_prof']; t = sum(p); print('   prof', [round(100*x/t,1) for x in p])
    else: print('$*', d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
run c3:64 MSW_K1_VARIANT=86
run c3:64 MSW_K1_VARIANT=104
run c3:64 MSW_K1_VARIANT=104 MSW_K1_RINGS=5,4
