#!/bin/bash
# fused stage form with epilogue warps (104-106): parity, then config 3 timing
o=gpurun_out/ag; mkdir -p $o
timeout 900 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "fused_layer_kernel" > $o/fused.log 2>&1; tail -3 $o/fused.log
nrun() { cases=$1; shift; env "$@" timeout 300 python tools/rom_sweep.py --cases $cases --steps 200 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
nrun c3:64 MSW_K1_VARIANT=86
nrun c3:64 MSW_K1_VARIANT=86 MSW_K1_RINGS=6,4
nrun c3:64 MSW_K1_VARIANT=104
nrun c3:64 MSW_K1_VARIANT=104 MSW_K1_RINGS=5,4
nrun c3:64 MSW_K1_VARIANT=104 MSW_K1_RINGS=5,3
nrun c3:64 MSW_K1_VARIANT=105
nrun c3:64 MSW_K1_VARIANT=106
nrun c3:64 MSW_K1_TUNE_LOG=1 2> $o/tune.log
nrun c3:1,c3:16,c2:16
