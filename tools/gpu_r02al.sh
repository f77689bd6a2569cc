#!/bin/bash
# 12/16-consumer-warp K-streaming instances with epilogue warps (104-106): parity, autotune at config 5
o=gpurun_out/al; mkdir -p $o
timeout 1200 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "every_k1_kernel_family or instability" > $o/family.log 2>&1; tail -3 $o/family.log
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 50 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
nrun c5:128 MSW_K1_VARIANT=104
nrun c5:128 MSW_K1_VARIANT=105
nrun c5:128 MSW_K1_VARIANT=95
nrun c5:32 MSW_K1_VARIANT=106
nrun c5:32 MSW_K1_VARIANT=95
nrun c5:32,c5:128 MSW_K1_TUNE_LOG=1 2> $o/tune.log
