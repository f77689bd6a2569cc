#!/bin/bash
# balanced cell work order: parity subset, A/B against the lexicographic table
o=gpurun_out/ak; mkdir -p $o
timeout 1200 python -m pytest tests/test_rom_gpu.py tests/test_fullsize_gpu.py -x -q -m gpu > $o/rom.log 2>&1; tail -3 $o/rom.log
export MSW_TUNE_CACHE=$PWD/$o/tune_cache.txt
nrun() { cases=$1; shift; env "$@" timeout 600 python tools/rom_sweep.py --cases $cases --steps 100 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print('ERR', l[:150]); continue
    if 'ms_step' in d: print('$*', d['config'], d['S'], round(d['ms_step'],4), round(d['k1_ms'],4), round(d['k2_ms'],4), d['k1']['k1_variant'], d['k1']['k1_source_tile'], d['k1']['k1_panel'], d['k1']['k1_rings'])
"; }
nrun c3:64,c5:1,c5:8,c5:32,c5:128,c3:16,c2:16
nrun c3:64,c5:1,c5:8,c5:32,c5:128,c3:16,c2:16 MSW_K1_ORDER=0
nrun c3:64,c5:32 
