#!/bin/bash
# epilogue-warp K-streaming instances, 256-bit operand loads: parity + cycle breakdown
o=gpurun_out/af; mkdir -p $o
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




















nrun() { cases=$1; shift; env "$@" timeout 300 python tools/rom_sweep.py --cases $cases --steps 30 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('noprof $*', d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }














run c5:128 MSW_K1_VARIANT=94
nrun c5:128 MSW_K1_VARIANT=103
nrun c5:128 MSW_K1_VARIANT=94
nrun c5:128 MSW_K1_VARIANT=99
nrun c5:32 MSW_K1_VARIANT=96
nrun c5:32 MSW_K1_VARIANT=100
