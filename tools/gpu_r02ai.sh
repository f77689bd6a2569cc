#!/bin/bash
# live-row-tile dispatch in the K-streaming k-loops: parity (family + instability + configs), config 5 sweep
o=gpurun_out/ai; mkdir -p $o
timeout 1200 python -m pytest tests/test_rom_gpu.py -x -q -m gpu -k "every_k1_kernel_family or instability or kstream" > $o/family.log 2>&1; tail -3 $o/family.log
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 30 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
nrun c5:128 MSW_K1_VARIANT=94
nrun c5:128 MSW_K1_VARIANT=42
nrun c5:32 MSW_K1_VARIANT=96
nrun c5:32 MSW_K1_VARIANT=39
nrun c5:1,c5:8,c5:32,c5:128 MSW_K1_TUNE_LOG=1 2> $o/tune.log
