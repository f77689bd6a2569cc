#!/bin/bash
# K-streaming instances with epilogue warps (94-98): parity, then config 5 S = 32 / 128 with cycle breakdown
o=gpurun_out/ae; mkdir -p $o
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "every_k1_kernel_family" > $o/family.log 2>&1; tail -3 $o/family.log
run() { cases=$1; shift; env "$@" MSW_LIB=$(realpath build/ab/lib_prof.so) MSW_K1_DEBUG=8 timeout 300 python tools/rom_sweep.py --cases $cases --steps 30 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'k1_prof' in d:
        p = d['k1_prof']; t = sum(p); print('   prof', [round(100*x/t,1) for x in p])
    else: print('$*', d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
run c5:128 MSW_K1_VARIANT=94
run c5:128 MSW_K1_VARIANT=94 MSW_K1_NP=16 MSW_K1_RINGS=4,3
run c5:128 MSW_K1_VARIANT=94 MSW_K1_NP=32 MSW_K1_RINGS=2,2
run c5:128 MSW_K1_VARIANT=97
run c5:128 MSW_K1_VARIANT=98
run c5:32 MSW_K1_VARIANT=95
run c5:32 MSW_K1_VARIANT=95 MSW_K1_NP=32
run c5:32 MSW_K1_VARIANT=96
run c5:32 MSW_K1_VARIANT=96 MSW_K1_NP=32
run c5:32 MSW_K1_VARIANT=97
run c5:32 MSW_K1_VARIANT=98
